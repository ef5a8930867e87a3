"""compat.install(): the REAL bridgegen (baseline/_ref or /root/reference)
with its ``_Machine._generic`` routed to libbgx.so.

CPU part: body classification on IR built by bridgegen itself, and the
reference's error behaviour (inconsistent extents, step budget) which is
raised before any device work.  GPU part: bridgegen's own API end to end —
its test suites' cases (test_interp.py:218-253, 301-339, test_einsum.py:
104-119, 169-202, test_acceptance.py:281-330) produce outputs bit-identical to
the reference's recorded outputs (tests/golden)."""

import os
import random
import sys

import numpy as np
import pytest

import _golden as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
bridgegen = G.import_bridgegen()   # hard failure, never a skip
from bridgegen import einsum, interp, intrinsics, ir  # noqa: E402
from bridgegen.gpu import register_gpu_intrinsics  # noqa: E402

from paper_2503_04771_b200 import compat, executor  # noqa: E402


@pytest.fixture
def registry():
    reg = intrinsics.default_registry()
    register_gpu_intrinsics(reg)
    return reg


def tv(x):
    x = np.asarray(x)
    return interp.TensorValue(ir.F64 if x.dtype == np.float64 else ir.F32, x.shape, x)


def generic_of(module):
    fn = module.lookup_symbol("einsum")
    return next(op for op in fn.regions[0].blocks[0].operations if op.name == "linalg.generic")


@pytest.mark.parametrize("text,n_in,kind", [
    ("(i,k),(k,j)->(i,j)", 2, "contract"), ("(i,j)->(j,i)", 1, "permute"),
    ("(i,j)->(i)", 1, "contract"), ("(i,j),(j,k),(k,l)->(i,l)", 3, "contract"),
    ("(i)->(i)", 1, "permute")])
def test_classify_reference_bodies(registry, text, n_in, kind):
    op = generic_of(einsum.build_einsum_function(registry, einsum.parse_einsum(text)))
    assert compat.classify_body(op.regions[0].blocks[0], n_in) == kind


def test_reference_errors_kept(registry):
    mod = einsum.build_einsum_function(registry, einsum.parse_einsum("(i,k),(k,j)->(i,j)"))
    with compat.backend():
        with pytest.raises(interp.InterpError, match="inconsistent extent"):
            interp.run_function(mod, "einsum", [tv(np.zeros((4, 3), np.float32)),
                                                tv(np.zeros((2, 5), np.float32)),
                                                tv(np.zeros((4, 5), np.float32))])
        z = np.zeros((256, 256), np.float32)
        with pytest.raises(interp.StepLimitExceeded, match="step budget of 10000000"):
            interp.run_function(mod, "einsum", [tv(z), tv(z), tv(z)])
    assert not compat.installed()


@pytest.mark.gpu
def test_reference_api_bit_exact_on_gpu(registry, dev):
    """Every golden case through bridgegen's own build/run API."""
    with compat.backend():
        for name, text, ins, init, want in G.generic_cases():
            elem = ir.F64 if want.dtype == np.float64 else ir.F32
            from bridgegen import fir
            mod = einsum.build_einsum_function(registry, einsum.parse_einsum(text),
                                               elem=fir.F64 if elem == ir.F64 else fir.F32)
            executor.reset_launch_log()
            [got] = interp.run_function(mod, "einsum", [tv(x) for x in ins] + [tv(init)],
                                        step_limit=10 ** 9)
            assert G.bits_equal(got.data, want), name
            assert executor.launch_log(), name


@pytest.mark.gpu
def test_reference_suite_replay_and_new_specs(registry, dev):
    """test_interp.py:301-339-style random specs with fresh seeds, bridgegen
    CPU evaluator vs the same call with the backend installed: bit-equal."""
    r = random.Random(4242)
    nr = np.random.default_rng(4242)
    letters = ["i", "j", "k", "l"]
    for _ in range(30):
        while True:
            ins = [tuple(r.sample(letters, r.randint(1, 3))) for _ in range(r.randint(1, 3))]
            used = sorted({x for t in ins for x in t})
            out = tuple(r.sample(used, r.randint(0, min(3, len(used)))))
            text = ",".join("(" + ",".join(t) + ")" for t in ins) + "->(" + ",".join(out) + ")"
            try:
                spec = einsum.parse_einsum(text)
                break
            except einsum.EinsumError:
                continue
        ext = {a: r.randint(1, 6) for a in spec.axes}
        arrs = [nr.standard_normal(tuple(ext[x] for x in t)).astype(np.float32) for t in spec.inputs]
        init = nr.standard_normal(tuple(ext[x] for x in spec.output)).astype(np.float32)
        mod = einsum.build_einsum_function(registry, spec)
        [ref] = interp.run_function(mod, "einsum", [tv(x) for x in arrs] + [tv(init)])
        with compat.backend():
            [got] = interp.run_function(mod, "einsum", [tv(x) for x in arrs] + [tv(init)])
        assert G.bits_equal(got.data, ref.data), text


@pytest.mark.gpu
def test_chained_generics_through_reference_builder(registry, dev):
    """test_einsum.py:169-202 — two generics in one bridgegen function."""
    from bridgegen import codegen
    from bridgegen.dialects import build_op
    spec = einsum.parse_einsum("(i,k),(k,j)->(i,j)")
    module = ir.IrModule(registry=registry.dialects)
    t = ir.TensorType(ir.F32, (None, None))
    region = module.new_region()
    build_op(registry.dialects, module, "func.func",
             attributes={"sym_name": ir.SymbolAttr("twice"),
                         "function_type": ir.TypeAttr(ir.FunctionType((t,) * 3, (t,)))},
             regions=[region])
    entry = module.append_block(region, [t] * 3)
    ctx = codegen.BuilderContext(module=module, registry=registry, region=region,
                                 entry_block=entry)
    ctx.set_block(entry)
    g1 = einsum.build_generic(ctx, registry, spec, list(entry.arguments))
    g2 = einsum.build_generic(ctx, registry, spec, [g1.results[0], entry.arguments[1],
                                                    entry.arguments[2]])
    ctx.build_op("func.return", [g2.results[0]])
    rng = np.random.default_rng(4)
    a = rng.random((3, 3)).astype(np.float32)
    b = rng.random((3, 3)).astype(np.float32)
    zero = np.zeros((3, 3), np.float32)
    [ref] = interp.run_function(module, "twice", [tv(a), tv(b), tv(zero)])
    with compat.backend():
        [got] = interp.run_function(module, "twice", [tv(a), tv(b), tv(zero)])
    assert G.bits_equal(got.data, ref.data)
    assert np.allclose(got.data, (a @ b) @ b, rtol=1e-4)


@pytest.mark.gpu
def test_schedule_string_attr_on_reference_op(registry, dev):
    """A ``bgx.schedule`` StringAttr on a real bridgegen linalg.generic pins the
    tensor-core tile (tf32 mode; the exact f32 default ignores schedules)."""
    mod = einsum.build_einsum_function(registry, einsum.parse_einsum("(i,k),(k,j)->(i,j)"))
    op = generic_of(mod)
    op.attributes["bgx.schedule"] = ir.StringAttr("tile_n=128,cta_group=1")
    rng = np.random.default_rng(9)
    a = rng.standard_normal((512, 256)).astype(np.float32)
    b = rng.standard_normal((256, 384)).astype(np.float32)
    c = np.zeros((512, 384), np.float32)
    with compat.backend("tf32"):
        executor.reset_launch_log()
        [got] = interp.run_function(mod, "einsum", [tv(a), tv(b), tv(c)], step_limit=10 ** 9)
    assert executor.tile_log() and executor.tile_log()[-1][:2] == (1, 128)
    want = a.astype(np.float64) @ b.astype(np.float64)
    assert np.linalg.norm(got.data - want) / np.linalg.norm(want) < 5e-3

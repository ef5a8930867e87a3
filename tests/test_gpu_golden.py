"""Parity gate: the reference's own einsum suites, run through this repo's
reference-shaped API on the B200, must reproduce the reference's outputs
BIT-FOR-BIT (tests/golden/generic_cases.npz was produced by bridgegen's
interp.run_function itself; see tests/golden/make_golden.py).

Covers test_interp.py:218-253, 301-339, test_einsum.py:104-119, 169-202,
test_acceptance.py:281-330 (criterion 8) and the extra BASELINE-pattern cases.
"""

import numpy as np
import pytest
import torch

import _golden as G
from paper_2503_04771_b200 import einsum as E
from paper_2503_04771_b200 import executor
from paper_2503_04771_b200 import interp as I

pytestmark = pytest.mark.gpu

CASES = G.generic_cases()


def _elem(arr):
    return E.F64 if arr.dtype == np.float64 else E.F32


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_reference_case_bit_exact(case, dev):
    name, text, ins, init, want = case
    spec = E.parse_einsum(text)
    elem = _elem(want)
    mod = E.build_einsum_function(None, spec, elem=elem)
    vals = [I.TensorValue(elem, x.shape, x) for x in ins] + [I.TensorValue(elem, init.shape, init)]
    init_before = init.copy()
    executor.reset_launch_log()
    [got] = I.run_function(mod, "einsum", vals, step_limit=None)
    assert G.bits_equal(got.data, want), (name, text, np.abs(got.data - want).max())
    assert np.array_equal(init, init_before)  # output operand untouched (interp.py:399)
    assert executor.launch_log(), "no bgx kernel launched"


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_reference_case_device_resident(case, dev):
    """Same cases with torch CUDA tensors in and out (no host round trip)."""
    name, text, ins, init, want = case
    spec = E.parse_einsum(text)
    elem = _elem(want)
    mod = E.build_einsum_function(None, spec, elem=elem)
    vals = [I.TensorValue(elem, x.shape, torch.from_numpy(np.ascontiguousarray(x)).to(dev))
            for x in (*ins, init)]
    [got] = I.run_function(mod, "einsum", vals, step_limit=None)
    assert got.data.is_cuda
    assert G.bits_equal(got.data.cpu().numpy(), want), name


def test_chained_generics_stay_on_device(dev):
    """test_einsum.py:169-202: two generics in one function, (a@b)@b."""
    byname = {c[0]: c for c in CASES}
    _, _, ins1, zero, _ = byname["einsum_chained_seed4_step1"]
    want = byname["einsum_chained_seed4_step2"][4]
    spec = E.parse_einsum("(i,k),(k,j)->(i,j)")
    module = E.Module()
    t2 = E.TensorType(E.F32, 2)
    ctx = E.FunctionBuilder(module, "twice", [t2] * 3)
    g1 = E.build_generic(ctx, None, spec, list(ctx.arguments))
    g2 = E.build_generic(ctx, None, spec, [g1.results[0], ctx.arguments[1], ctx.arguments[2]])
    ctx.ret([g2.results[0]])
    text = E.print_module(module)
    assert "%0 = linalg.generic" in text and "%6 = linalg.generic" in text
    a, b = ins1
    executor.reset_launch_log()
    [out] = I.run_function(module, "twice", [I.TensorValue(E.F32, x.shape, x) for x in (a, b, zero)])
    assert G.bits_equal(out.data, want)
    # two device launches, no host round trip (tiny operands: the skinny
    # exact GEMM rule may pick the loop nest instead of SIMT tiles)
    log = executor.launch_log()
    assert len(log) == 2 and set(log) <= {"simt-exact", "generic"}, log


def test_modes_agree_within_tolerance(dev):
    """ffma / tensor-core modes vs the bit-exact result (rtol 1e-5 for FFMA)."""
    rng = np.random.default_rng(3)
    a = rng.standard_normal((70, 90)).astype(np.float32)
    b = rng.standard_normal((90, 50)).astype(np.float32)
    c = np.zeros((70, 50), np.float32)
    mod = E.build_einsum_function(None, E.parse_einsum("(i,k),(k,j)->(i,j)"))
    vals = [I.TensorValue(E.F32, x.shape, x) for x in (a, b, c)]
    [exact] = I.run_function(mod, "einsum", vals, mode="exact")
    [ffma] = I.run_function(mod, "einsum", vals, mode="ffma")
    den = np.linalg.norm(exact.data)
    assert np.linalg.norm(ffma.data - exact.data) / den <= 1e-5

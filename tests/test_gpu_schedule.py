"""Schedules (transform-style tiling parameters) attached to a
generic op: they reach kernel selection and never change results beyond the
tolerance of the chosen path."""

import numpy as np
import pytest
import torch

from paper_2503_04771_b200 import einsum as E
from paper_2503_04771_b200 import executor
from paper_2503_04771_b200 import interp as I
from paper_2503_04771_b200.api import contract
from paper_2503_04771_b200.schedule import Schedule

pytestmark = pytest.mark.gpu

MM = "(i,k),(k,j)->(i,j)"


def _relf(got, want):
    got, want = got.double(), want.double()
    return float((got - want).norm() / want.norm())


@pytest.mark.parametrize("sched,expect", [
    ("cta_group=1,tile_n=128", (1, 128)),
    ("cta_group=1,tile_n=64", (1, 64)),
    ("cta_group=2,tile_n=256,raster=-4", (2, 256)),
    ("cta_group=2,tile_n=512,stages=3", (2, 512)),
    ("cta_group=2,tile_n=128,max_ctas=16", (2, 128)),
])
def test_schedule_on_op_selects_tile(dev, sched, expect):
    g = torch.Generator(device=dev).manual_seed(7)
    a = torch.randn(512, 1024, device=dev, generator=g).bfloat16()
    b = torch.randn(1024, 1024, device=dev, generator=g).bfloat16()
    c = torch.zeros(512, 1024, device=dev, dtype=torch.bfloat16)
    mod = E.build_einsum_function(None, E.parse_einsum(MM), elem=E.BF16, schedule=sched)
    executor.reset_launch_log()
    [got] = I.run_function(mod, "einsum", [I.TensorValue(E.BF16, x.shape, x) for x in (a, b, c)],
                              step_limit=None)
    cg, bn, _ = executor.tile_log()[-1]
    assert (cg, bn) == expect
    assert executor.launch_log()[0].startswith("tcgen05")
    assert _relf(got.data, a.double() @ b.double()) < 1e-2


def test_schedule_argument_overridden_by_op(dev):
    a = torch.randn(256, 512, device=dev).half()
    b = torch.randn(512, 768, device=dev).half()
    c = torch.zeros(256, 768, device=dev, dtype=torch.float16)
    mod = E.build_einsum_function(None, E.parse_einsum(MM), elem=E.F16,
                                  schedule=Schedule(cta_group=1, tile_n=256))
    executor.reset_launch_log()
    I.run_function(mod, "einsum", [I.TensorValue(E.F16, x.shape, x) for x in (a, b, c)],
                   schedule="cta_group=2,tile_n=128", step_limit=None)
    assert executor.tile_log()[-1][:2] == (1, 256)
    # no schedule on the op: the call's schedule applies
    mod2 = E.build_einsum_function(None, E.parse_einsum(MM), elem=E.F16)
    executor.reset_launch_log()
    I.run_function(mod2, "einsum", [I.TensorValue(E.F16, x.shape, x) for x in (a, b, c)],
                   schedule="cta_group=2,tile_n=128", step_limit=None)
    assert executor.tile_log()[-1][:2] == (2, 128)


def test_schedule_split_k_through_contract(dev):
    a = torch.randn(256, 65536, device=dev).bfloat16()
    b = torch.randn(65536, 256, device=dev).bfloat16()
    executor.reset_launch_log()
    y = contract(MM, a, b, schedule="splits=4,cta_group=1,tile_n=128")
    assert executor.launch_log() == ["tcgen05-splitk"]
    assert executor.tile_log()[-1] == (1, 128, 4)
    assert _relf(y, a.double() @ b.double()) < 1e-2


def test_schedule_ignored_by_exact_fp32_path(dev):
    """f32 in 'auto' mode is the bit-exact SIMT path: a schedule does not
    change which kernel runs nor a single bit of the result."""
    rng = np.random.default_rng(3)
    a, b = rng.random((33, 17), np.float32), rng.random((17, 29), np.float32)
    c = np.zeros((33, 29), np.float32)
    mod = E.build_einsum_function(None, E.parse_einsum(MM))
    mods = E.build_einsum_function(None, E.parse_einsum(MM), schedule="cta_group=2,tile_n=512")
    vals = [I.TensorValue(E.F32, x.shape, x) for x in (a, b, c)]
    [r0] = I.run_function(mod, "einsum", vals)
    [r1] = I.run_function(mods, "einsum", vals)
    assert np.array_equal(np.asarray(r0.data).view(np.uint32), np.asarray(r1.data).view(np.uint32))

"""Maximum sizes (SURVEY §8c edge cases): operands and outputs with more than
2^31 elements, so every kernel's flat / row / tile indexing has to be 64-bit.
Permutations and copies are checked bit for bit against torch's own copy;
the exact row reduction against the reference's sequential order on sampled
rows; the tensor-core GEMM against an f32 product on sampled rows (bf16
tolerance 1e-2, north_star)."""

import numpy as np
import pytest
import torch

from paper_2503_04771_b200 import contract

pytestmark = pytest.mark.gpu

BIG = (1 << 31) + (1 << 20)   # just past 2^31 elements


def _fill(shape, dtype, dev, seed):
    g = torch.Generator(device=dev).manual_seed(seed)
    return torch.randn(shape, generator=g, device=dev, dtype=torch.float32).to(dtype)


def test_transpose_past_2_31(dev):
    x = _fill((65536, 32784), torch.bfloat16, dev, 1)       # 2.149e9 elements
    assert x.numel() > 1 << 31
    got = contract("(i,j)->(j,i)", x)
    assert torch.equal(got, x.t().contiguous())


def test_3d_permute_past_2_31(dev):
    x = _fill((1024, 2049, 1024), torch.bfloat16, dev, 2)
    assert x.numel() > 1 << 31
    got = contract("(a,b,c)->(c,b,a)", x)
    assert torch.equal(got, x.permute(2, 1, 0).contiguous())


def test_identity_copy_past_2_31(dev):
    x = _fill((BIG,), torch.bfloat16, dev, 3)
    got = contract("(i)->(i)", x)
    assert torch.equal(got, x)


def test_short_rows_copy_past_2_31(dev):
    # inner rows of 96 elements moved as a unit ((a,b,c)->(b,a,c)): the
    # short-row copy kernel's 32-bit flat index must hand over to 64-bit
    x = _fill((16384, 1366, 96), torch.bfloat16, dev, 4)
    assert x.numel() > 1 << 31
    got = contract("(a,b,c)->(b,a,c)", x)
    assert torch.equal(got, x.permute(1, 0, 2).contiguous())


def test_exact_row_reduction_past_2_31(dev):
    x = _fill((65600, 32768), torch.float32, dev, 5)       # 2.15e9 elements, 8.6 GB
    got = contract("(i,j)->(i)", x)
    for r in (0, 1, 31337, 65599):
        row = x[r].cpu().numpy()
        want = np.add.accumulate(np.concatenate([[np.float32(0)], row]), dtype=np.float32)[-1]
        assert got[r].item() == float(want), r   # the reference's order, bit for bit


def test_gemm_output_past_2_31(dev):
    a = _fill((65536, 64), torch.bfloat16, dev, 6)
    b = _fill((64, 32784), torch.bfloat16, dev, 7)
    got = contract("(i,k),(k,j)->(i,j)", a, b)             # 2.149e9 outputs
    assert got.numel() > 1 << 31
    for r in (0, 40000, 65535):
        want = a[r:r + 1].float() @ b.float()
        err = ((got[r:r + 1].float() - want).norm() / want.norm()).item()
        assert err <= 1e-2, (r, err)
    # the last columns of the last row (the highest flat offsets)
    want = a[-1:].float() @ b[:, -64:].float()
    err = ((got[-1:, -64:].float() - want).norm() / want.norm()).item()
    assert err <= 1e-2


@pytest.mark.parametrize("text,dtype,mode", [
    ("(i,j)->()", torch.float32, "ffma"),          # tree: contiguous, full reduction
    ("(i,j)->(i)", torch.float32, "ffma"),         # tree: contiguous rows
    ("(i,j)->(j)", torch.float32, "ffma"),         # tree: column reduction
    ("(i,j)->(j)", torch.bfloat16, "auto"),        # tree: 16-bit columns, two per lane
])
def test_tree_reductions_past_2_31(dev, text, dtype, mode):
    x = _fill((65600, 32768), dtype, dev, 8)
    assert x.numel() > 1 << 31
    got = contract(text, x, mode=mode).double()
    dims = {"(i,j)->()": (0, 1), "(i,j)->(i)": (1,), "(i,j)->(j)": (0,)}[text]
    want = x.double().sum(dim=dims)
    scale = want.abs().max().item() + x.shape[dims[0]] ** 0.5
    err = (got - want).abs().max().item() / scale
    assert err <= (2e-2 if dtype == torch.bfloat16 else 1e-4), err

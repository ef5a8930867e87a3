"""bgx_permute on the B200: bit-exact against numpy transposition (which the
oracle tests pin to the reference's passthrough body, einsum.py:105-108),
including IEEE specials, every element size, strided views, ragged extents
and the BASELINE C2 sizes (8192^2 and 256x512x512 f32)."""

import numpy as np
import pytest
import torch

from paper_2503_04771_b200 import contract, executor

pytestmark = pytest.mark.gpu


def letters(n):
    return "abcdefgh"[:n]


def spec_for(perm):
    src = letters(len(perm))
    dst = "".join(src[p] for p in perm)
    return f"({','.join(src)})->({','.join(dst)})"


@pytest.mark.parametrize("shape,perm", [
    ((64, 64), (1, 0)),
    ((8192, 8192), (1, 0)),
    ((256, 512, 512), (2, 1, 0)),
    ((5, 33, 7), (2, 0, 1)),
    ((3, 4, 5, 6), (3, 1, 0, 2)),
    ((2, 3, 4, 5, 6, 7), (5, 4, 3, 2, 1, 0)),
    ((37,), (0,)),
    ((129, 67), (0, 1)),
    ((1, 1000, 1), (2, 1, 0)),
    ((4, 1, 130, 3), (2, 0, 3, 1)),
])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64, torch.bfloat16, torch.float16])
def test_permute_bit_exact(dev, shape, perm, dtype):
    g = torch.Generator().manual_seed(0)
    x = torch.randn(shape, generator=g).to(dtype)
    out = contract(spec_for(perm), x.to(dev))
    want = x.permute(*perm).contiguous()
    bits = lambda t: t.contiguous().reshape(-1).view(torch.uint8)  # noqa: E731
    assert tuple(out.shape) == tuple(want.shape)
    assert torch.equal(bits(out.cpu()), bits(want))


def test_permute_ieee_specials_bits(dev):
    bits = np.array([0x7F800000, 0xFF800000, 0x80000000, 0x00000001, 0x7FC00001,
                     0x7F800001, 0x3F800000, 0x00800000], dtype=np.uint32)
    x = np.tile(bits, 64 * 8).reshape(64, 64).view(np.float32)
    y = contract("(i,j)->(j,i)", torch.from_numpy(x).to(dev)).cpu().numpy()
    assert np.array_equal(y.view(np.uint32), x.T.view(np.uint32))  # sNaN payload kept


def test_permute_strided_views(dev):
    base = torch.randn(40, 70, device=dev)
    view = base[3:35:2, 5:65:3]           # non-contiguous input
    out = torch.empty(20, 16, device=dev)
    executor.permute(view, out, (1, 0))
    assert torch.equal(out, view.t().contiguous())
    dst = torch.zeros(32, 60, device=dev)
    target = dst[::2, 1:41:2]             # strided output, same shape as view
    executor.permute(view, target, (0, 1))
    assert torch.equal(target, view)


def test_permute_empty(dev):
    x = torch.empty(0, 5, device=dev)
    out = contract("(i,j)->(j,i)", x)
    assert out.shape == (5, 0)

"""Performance floors (generous, power-cap tolerant) so that a regression in
a later change shows up in `pytest -m gpu`, not only in bench.py: the
headline GEMM shape, BASELINE config 4, and the config-2 permutation."""

import statistics

import pytest
import torch

from paper_2503_04771_b200.api import contract

pytestmark = pytest.mark.gpu


def _ms(fn, iters=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(iters)]
    for s, e in ev:
        s.record()
        fn()
        e.record()
    torch.cuda.synchronize()
    return statistics.median(s.elapsed_time(e) for s, e in ev)


@pytest.mark.parametrize("M,N,K,floor", [(16384, 8192, 8192, 1100.0), (4096, 4096, 4096, 1000.0)])
def test_gemm_floor(dev, M, N, K, floor):
    a = torch.randn(M, K, device=dev).bfloat16()
    b = torch.randn(K, N, device=dev).bfloat16()
    out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    ms = _ms(lambda: contract("(i,k),(k,j)->(i,j)", a, b, out=out))
    tflops = 2 * M * N * K / ms / 1e9
    assert tflops >= floor, f"{M}x{N}x{K}: {tflops:.0f} TFLOP/s < {floor}"


def test_permute_floor(dev):
    x = torch.randn(8192, 8192, device=dev)
    out = torch.empty(8192, 8192, device=dev)
    ms = _ms(lambda: contract("(i,j)->(j,i)", x, out=out))
    gbs = 2 * x.numel() * 4 / ms / 1e6
    assert gbs >= 4000.0, f"transpose {gbs:.0f} GB/s < 4000"


@pytest.mark.parametrize("spec,shape", [("(i,j)->(i,j)", (8192, 8192)),
                                        ("(i)->(i)", (1 << 26,)),
                                        ("(i,j,k)->(i,j,k)", (64, 1024, 1024))])
def test_identity_copy_floor(dev, spec, shape):
    """Passthrough bodies whose dims all merge into one contiguous run (round
    2 fix: that run was copied by ONE block, ~53 GB/s) spread over every SM."""
    x = torch.randn(shape, device=dev)
    out = torch.empty_like(x)
    ms = _ms(lambda: contract(spec, x, out=out))
    gbs = 2 * x.numel() * 4 / ms / 1e6
    assert torch.equal(out, x)
    assert gbs >= 3000, f"{spec}: {gbs:.0f} GB/s"


@pytest.mark.parametrize("n", [1, 7, 4095, 4097, 1 << 20, (1 << 20) + 3])
def test_long_row_copy_chunks_exact(dev, n):
    """Chunked row copies: every element lands once, vector and scalar paths."""
    x = torch.randn(n, device=dev)
    assert torch.equal(contract("(i)->(i)", x), x)
    y = torch.randn(3, n, device=dev)[:, : max(1, n - 1)]     # unaligned rows: scalar path
    assert torch.equal(contract("(b,i)->(b,i)", y), y)


@pytest.mark.parametrize("spec,shapes,ceiling_ms", [
    ("(i,k),(k)->(i)", [(8192, 8192), (8192,)], 0.25),             # exact GEMV (row-reduction kernel), ~0.09 ms
    ("(i,k)->(i)", [(8192, 8192)], 0.25),                           # exact row sums, ~0.08 ms
    ("(a),(b,c,d)->()", [(4,), (64, 256, 256)], 150.0),             # block-per-output chain, ~47 ms (was ~470)
    ("(d,a,c),(c,d,b)->(b,c,d)", [(256, 64, 64), (64, 256, 256)], 60.0),  # walk order + invariant hoist
])
def test_exact_generic_ceilings(dev, spec, shapes, ceiling_ms):
    """Exact (reference-order) generic bodies: generous time ceilings on the
    round-2 kernel paths, so a planner or kernel regression fails here."""
    xs = [torch.randn(s, device=dev) for s in shapes]
    ms = _ms(lambda: contract(spec, *xs), iters=3)
    assert ms <= ceiling_ms, f"{spec}: {ms:.2f} ms > {ceiling_ms}"

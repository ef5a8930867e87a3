"""Contraction kernels on the B200 vs the CPU oracle.

* SIMT exact (f32): bit-identical to the reference's arithmetic (oracle
  gemm_kseq, itself pinned to bridgegen by tests/test_oracle.py), incl. the
  BASELINE C1 config (256^3 f32 via the DSL).
* tcgen05 (bf16/f16 in, f32 accumulate): relative Frobenius error <= 1e-2
  (north_star tolerance) against the oracle on the bf16-rounded inputs, for
  every operand layout (A K-/M-major x B K-/N-major), batch, beta (c0), ragged
  M/N/K and each output dtype; plus row-sampled parity at the BASELINE C3/C4
  sizes.
"""

import numpy as np
import pytest
import torch

import oracle
from paper_2503_04771_b200 import _lib, contract, executor
from paper_2503_04771_b200 import einsum as E
from paper_2503_04771_b200 import interp as I

pytestmark = pytest.mark.gpu

BF16_TOL = 1e-2
FFMA_TOL = 1e-5


def rnd(shape, seed, dev, dtype=torch.float32):
    x = np.random.default_rng(seed).standard_normal(shape, dtype=np.float32)
    return torch.from_numpy(x).to(dev).to(dtype)


def np32(t):
    return t.float().cpu().numpy()


def test_c1_fp32_256_cubed_bit_exact(dev):
    """BASELINE config 1 through the DSL: (i,j),(j,k)->(i,k) f32 256^3."""
    rng = np.random.default_rng(1)
    a = rng.standard_normal((256, 256), dtype=np.float32)
    b = np.random.default_rng(2).standard_normal((256, 256), dtype=np.float32)
    c = np.zeros((256, 256), np.float32)
    mod = E.build_einsum_function(None, E.parse_einsum("(i,j),(j,k)->(i,k)"))
    executor.reset_launch_log()
    [got] = I.run_function(mod, "einsum", [I.TensorValue(E.F32, x.shape, x) for x in (a, b, c)],
                           step_limit=None)
    assert np.array_equal(got.data, oracle.gemm_kseq(a, b, c))
    assert executor.launch_log() == ["simt-exact"]


def test_step_limit_mirrors_reference(dev):
    """256^3 needs 50,331,650 reference steps: the default
    budget of 10^7 raises StepLimitExceeded exactly like the reference."""
    mod = E.build_einsum_function(None, E.parse_einsum("(i,j),(j,k)->(i,k)"))
    z = np.zeros((256, 256), np.float32)
    with pytest.raises(I.StepLimitExceeded, match="step budget of 10000000"):
        I.run_function(mod, "einsum", [I.TensorValue(E.F32, z.shape, z)] * 3)
    I.run_function(mod, "einsum", [I.TensorValue(E.F32, z.shape, z)] * 3, step_limit=50_331_650)
    with pytest.raises(I.StepLimitExceeded):
        I.run_function(mod, "einsum", [I.TensorValue(E.F32, z.shape, z)] * 3,
                       step_limit=50_331_649)


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (7, 5, 3), (64, 64, 64), (130, 70, 300)])
@pytest.mark.parametrize("beta", [False, True])
def test_fp32_exact_and_ffma(dev, M, N, K, beta):
    a, b = rnd((M, K), 1, dev), rnd((K, N), 2, dev)
    c0 = rnd((M, N), 3, dev) if beta else None
    ex = contract("(i,k),(k,j)->(i,j)", a, b, c0=c0, mode="exact")
    want = oracle.gemm_kseq(np32(a), np32(b), np32(c0) if beta else None)
    assert np.array_equal(np32(ex), want)
    ff = contract("(i,k),(k,j)->(i,j)", a, b, c0=c0, mode="ffma")
    assert oracle.rel_frobenius(np32(ff), want) <= FFMA_TOL


@pytest.mark.parametrize("M,N,K", [(256, 256, 256), (332, 260, 132), (250, 300, 36),
                                   (256, 256, 1000), (64, 1024, 256)])
@pytest.mark.parametrize("beta", [False, True])
def test_fp32_exact_small_cp_path(dev, M, N, K, beta):
    """Latency-bound row-major f32 (the cp.async ring kernel): ragged M/N, K
    tails shorter than a stage, c0 — bit-identical to the reference order."""
    a, b = rnd((M, K), 11, dev), rnd((K, N), 12, dev)
    c0 = rnd((M, N), 13, dev) if beta else None
    ex = contract("(i,k),(k,j)->(i,j)", a, b, c0=c0, mode="exact")
    want = oracle.gemm_kseq(np32(a), np32(b), np32(c0) if beta else None)
    assert np.array_equal(np32(ex), want)
    ff = contract("(i,k),(k,j)->(i,j)", a, b, c0=c0, mode="ffma")
    assert oracle.rel_frobenius(np32(ff), want) <= FFMA_TOL


def test_f64_exact(dev):
    a = rnd((33, 41), 4, dev, torch.float64)
    b = rnd((41, 19), 5, dev, torch.float64)
    got = contract("(i,k),(k,j)->(i,j)", a, b).cpu().numpy()
    want = oracle.generic([("i", "k"), ("k", "j")], ("i", "j"),
                          [a.cpu().numpy(), b.cpu().numpy()], np.zeros((33, 19)))
    assert np.array_equal(got, want)


LAYOUTS = {
    # spec, how to build A and B so that A is K- or M-major and B K- or N-major
    "A_k_B_n": "(i,k),(k,j)->(i,j)",
    "A_m_B_n": "(k,i),(k,j)->(i,j)",
    "A_k_B_k": "(i,k),(j,k)->(i,j)",
    "A_m_B_k": "(k,i),(j,k)->(i,j)",
}


@pytest.mark.parametrize("layout", list(LAYOUTS))
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 512, 640), (200, 136, 72), (1000, 520, 1000)])
@pytest.mark.parametrize("cta_group,tile_n", [(1, 0), (2, 0), (2, 512)])
def test_tcgen05_layouts(dev, layout, dtype, M, N, K, cta_group, tile_n):
    spec = E.parse_einsum(LAYOUTS[layout])
    shp = {"i": M, "j": N, "k": K}
    a = rnd(tuple(shp[x] for x in spec.inputs[0]), 11, dev, dtype)
    b = rnd(tuple(shp[x] for x in spec.inputs[1]), 12, dev, dtype)
    executor.reset_launch_log()
    out = contract(spec, a, b, out_dtype=torch.float32, mode="tc",
                   schedule={"cta_group": cta_group, "tile_n": tile_n})
    assert [k.split("-")[0] for k in executor.launch_log()] == ["tcgen05"]
    A = np32(a) if spec.inputs[0] == ("i", "k") else np32(a).T
    B = np32(b) if spec.inputs[1] == ("k", "j") else np32(b).T
    want = oracle.gemm_kseq(np.ascontiguousarray(A), np.ascontiguousarray(B))
    err = oracle.rel_frobenius(np32(out), want)
    assert err <= BF16_TOL, err
    # tf32-free f32 accumulation should be far tighter than the bar
    assert err <= 1e-5, err


@pytest.mark.parametrize("tile_n", [64, 128, 256, 512])
@pytest.mark.parametrize("cta_group", [1, 2])
def test_tcgen05_tile_sizes_and_bf16_out(dev, tile_n, cta_group):
    a, b = rnd((384, 320), 21, dev, torch.bfloat16), rnd((320, 1088), 22, dev, torch.bfloat16)
    c0 = rnd((384, 1088), 23, dev, torch.bfloat16)
    out = contract("(i,k),(k,j)->(i,j)", a, b, c0=c0, mode="tc",
                   schedule={"tile_n": tile_n, "cta_group": cta_group})
    assert out.dtype == torch.bfloat16
    want = oracle.gemm_kseq(np32(a), np32(b), np32(c0))
    assert oracle.rel_frobenius(np32(out), want) <= BF16_TOL


def test_tcgen05_batched_c3_pattern(dev):
    """(b,i,j),(b,j,k)->(b,i,k), batch folded into the tile scheduler."""
    a, b = rnd((5, 192, 160), 31, dev, torch.bfloat16), rnd((5, 160, 272), 32, dev, torch.bfloat16)
    executor.reset_launch_log()
    out = contract("(b,i,j),(b,j,k)->(b,i,k)", a, b, out_dtype=torch.float32)
    assert [k.split("-")[0] for k in executor.launch_log()] == ["tcgen05"]
    want = oracle.gemm_kseq(np32(a), np32(b))
    assert oracle.rel_frobenius(np32(out), want) <= 1e-5


def test_tcgen05_output_transposed(dev):
    """(i,k),(k,j)->(j,i): the planner swaps operand roles so the output's
    unit-stride index is N."""
    a, b = rnd((300, 200), 41, dev, torch.bfloat16), rnd((200, 176), 42, dev, torch.bfloat16)
    out = contract("(i,k),(k,j)->(j,i)", a, b, out_dtype=torch.float32)
    want = oracle.gemm_kseq(np32(a), np32(b)).T
    assert oracle.rel_frobenius(np32(out), want) <= 1e-5


@pytest.mark.parametrize("cfg", ["c3", "c4"])
def test_baseline_sizes_row_sampled(dev, cfg):
    """BASELINE C3 (64 x 1024^3) and C4 (4096^3) bf16: full GPU run, oracle on
    sampled rows of every batch (ladder L1/L2 of SURVEY §8c)."""
    if cfg == "c3":
        a, b = rnd((64, 1024, 1024), 1, dev, torch.bfloat16), rnd((64, 1024, 1024), 2, dev, torch.bfloat16)
        spec = "(b,i,j),(b,j,k)->(b,i,k)"
    else:
        a, b = rnd((4096, 4096), 1, dev, torch.bfloat16), rnd((4096, 4096), 2, dev, torch.bfloat16)
        spec = "(i,k),(k,j)->(i,j)"
    out = contract(spec, a, b)
    assert out.dtype == torch.bfloat16
    rows = np.random.default_rng(9).choice(a.shape[-2], 8, replace=False)
    A, B, O = np32(a), np32(b), np32(out)
    if cfg == "c4":
        A, B, O = A[None], B[None], O[None]
    for bi in range(0, A.shape[0], max(1, A.shape[0] // 4)):
        want = oracle.gemm_kseq(np.ascontiguousarray(A[bi][rows]), B[bi])
        assert oracle.rel_frobenius(O[bi][rows], want) <= BF16_TOL
    assert np.isfinite(O).all()


def test_contract_kernel_selection(dev):
    a = rnd((256, 256), 1, dev, torch.bfloat16)
    d = _lib.BgxContractDesc()
    d.batch, d.M, d.N, d.K = 1, 256, 256, 256
    d.a = d.b = a.data_ptr()
    d.out = a.data_ptr()
    d.a_stride[:] = [0, 256, 1]
    d.b_stride[:] = [0, 256, 1]
    d.o_stride[:] = [0, 256, 1]
    d.in_dtype = d.out_dtype = _lib.BF16
    assert _lib.load().bgx_contract_kernel(d) == _lib.KERNEL_TC
    d.a_stride[:] = [0, 255, 1]  # 510-byte rows: not TMA legal
    assert _lib.load().bgx_contract_kernel(d) == _lib.KERNEL_SIMT16
    d.mode = _lib.MODE_TC
    assert _lib.load().bgx_contract_kernel(d) == _lib.ERR_UNSUPPORTED


def test_tile_choice_abi(dev):
    """bgx_contract_tile reports the wave-quantisation-driven tile choice."""
    import ctypes
    a = rnd((8, 8), 1, dev, torch.bfloat16)
    d = _lib.BgxContractDesc()
    d.a = d.b = d.out = a.data_ptr()
    d.in_dtype = d.out_dtype = _lib.BF16
    cg, bn = ctypes.c_int32(), ctypes.c_int32()
    for (M, N, K) in [(4096, 4096, 4096), (32768, 8192, 8192), (256, 64, 4096)]:
        d.batch, d.M, d.N, d.K = 1, M, N, K
        d.a_stride[:] = [0, K, 1]
        d.b_stride[:] = [0, N, 1]
        d.o_stride[:] = [0, N, 1]
        assert _lib.load().bgx_contract_tile(d, cg, bn) == 0
        assert cg.value in (1, 2) and bn.value in (64, 128, 256, 512)


@pytest.mark.parametrize("out_dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("cta_group", [1, 2])
def test_tcgen05_unaligned_output_uses_direct_stores(dev, out_dtype, cta_group):
    """N = 100 (200-byte bf16 rows): no TMA map for the output, so the
    epilogue falls back to direct stores; B is K-major so TC stays legal."""
    a, b = rnd((200, 64), 51, dev, torch.bfloat16), rnd((100, 64), 52, dev, torch.bfloat16)
    executor.reset_launch_log()
    out = contract("(i,k),(j,k)->(i,j)", a, b, out_dtype=out_dtype, mode="tc",
                   schedule={"cta_group": cta_group})
    assert [k.split("-")[0] for k in executor.launch_log()] == ["tcgen05"]
    want = oracle.gemm_kseq(np32(a), np.ascontiguousarray(np32(b).T))
    assert oracle.rel_frobenius(np32(out), want) <= BF16_TOL


@pytest.mark.parametrize("M,N,K,batch", [(256, 256, 16384, 1), (200, 136, 9000, 1), (128, 256, 4096, 3)])
@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_splitk_matches_oracle(dev, M, N, K, batch, out_dtype):
    """Small-output / long-K contractions split K across SMs (f32 partials +
    in-order reduction); forced split counts and the automatic plan."""
    a = rnd((batch, M, K), 61, dev, torch.bfloat16)
    b = rnd((batch, K, N), 62, dev, torch.bfloat16)
    c0 = rnd((batch, M, N), 63, dev, out_dtype)
    want = oracle.gemm_kseq(np32(a), np32(b), np32(c0))
    for sched in (None, {"splits": 3}, {"splits": 7, "cta_group": 2}):
        executor.reset_launch_log()
        out = contract("(b,i,k),(b,k,j)->(b,i,j)", a, b, c0=c0, out_dtype=out_dtype, schedule=sched)
        log = executor.launch_log()
        if sched:
            assert log == ["tcgen05-splitk"], log
        err = oracle.rel_frobenius(np32(out), want)
        assert err <= (1e-5 if out_dtype == torch.float32 else BF16_TOL), (sched, err)


def test_splitk_plan_only_for_small_outputs(dev):
    import ctypes
    a = rnd((8, 8), 1, dev, torch.bfloat16)
    d = _lib.BgxContractDesc()
    d.a = d.b = d.out = a.data_ptr()
    d.in_dtype = d.out_dtype = _lib.BF16
    sp, ws = ctypes.c_int32(), ctypes.c_int64()
    for (M, N, K, expect) in [(256, 256, 1 << 20, True), (8192, 8192, 8192, False)]:
        d.batch, d.M, d.N, d.K = 1, M, N, K
        d.a_stride[:] = [0, K, 1]
        d.b_stride[:] = [0, N, 1]
        d.o_stride[:] = [0, N, 1]
        assert _lib.load().bgx_contract_splitk_plan(d, sp, ws) == 0
        assert (sp.value > 1) == expect and (ws.value > 0) == expect


TF32_TOL = 5e-3   # 10-bit mantissa products, f32 accumulation


@pytest.mark.parametrize("layout", list(LAYOUTS))
@pytest.mark.parametrize("cta_group,tile_n", [(1, 0), (2, 0), (2, 512)])
@pytest.mark.parametrize("M,N,K", [(128, 256, 96), (1000, 520, 1000)])
def test_tf32_tensor_cores(dev, layout, cta_group, tile_n, M, N, K):
    """f32 inputs on tcgen05 kind::tf32 (opt-in mode='tf32')."""
    spec = E.parse_einsum(LAYOUTS[layout])
    shp = {"i": M, "j": N, "k": K}
    a = rnd(tuple(shp[x] for x in spec.inputs[0]), 71, dev)
    b = rnd(tuple(shp[x] for x in spec.inputs[1]), 72, dev)
    executor.reset_launch_log()
    out = contract(spec, a, b, mode="tf32", schedule={"cta_group": cta_group, "tile_n": tile_n})
    # MN-major operands are first made K-major by bgx_permute (tf32 kernel limit)
    assert [k.split("-")[0] for k in executor.launch_log() if k != "permute"] == ["tcgen05"]
    A = np32(a) if spec.inputs[0] == ("i", "k") else np32(a).T
    B = np32(b) if spec.inputs[1] == ("k", "j") else np32(b).T
    want = oracle.gemm_kseq(np.ascontiguousarray(A), np.ascontiguousarray(B))
    err = oracle.rel_frobenius(np32(out), want)
    assert 1e-7 < err <= TF32_TOL, err   # tf32 really is lower precision than f32 FFMA


def test_tf32_c1_config_and_splitk(dev):
    a, b = rnd((256, 256), 1, dev), rnd((256, 256), 2, dev)
    out = contract("(i,j),(j,k)->(i,k)", a, b, mode="tf32")
    assert oracle.rel_frobenius(np32(out), oracle.gemm_kseq(np32(a), np32(b))) <= TF32_TOL
    a, b = rnd((128, 65536), 3, dev), rnd((65536, 128), 4, dev)
    executor.reset_launch_log()
    out = contract("(i,k),(k,j)->(i,j)", a, b, mode="tf32")
    assert [k for k in executor.launch_log() if k != "permute"] == ["tcgen05-splitk"]
    ref = oracle.gemm_kseq(np32(a), np32(b))
    assert oracle.rel_frobenius(np32(out), ref) <= TF32_TOL


@pytest.mark.parametrize("M,N,K,bn", [(2304, 2560, 2048, 0), (4096, 4096, 4096, 0),
                                      (4096, 4608, 1024, 512), (2816, 3072, 8192, 512)])
def test_tail_split_matches_unsplit(dev, M, N, K, bn):
    """Stream-K-style tail split: only the last partial wave's tiles are split
    in K; results match the unsplit kernel to f32 summation-order noise and
    the oracle on sampled rows."""
    a, b = rnd((M, K), 81, dev, torch.bfloat16), rnd((K, N), 82, dev, torch.bfloat16)
    c0 = rnd((M, N), 83, dev, torch.float32)
    tile = {"tile_n": bn, "cta_group": 2} if bn else {}
    executor.reset_launch_log()
    tail = contract("(i,k),(k,j)->(i,j)", a, b, c0=c0, out_dtype=torch.float32,
                    schedule=dict(tile, splits=-2))
    assert executor.launch_log() == ["tcgen05-tailsplit"], executor.launch_log()
    plain = contract("(i,k),(k,j)->(i,j)", a, b, c0=c0, out_dtype=torch.float32,
                     schedule=dict(tile, no_splitk=1))
    assert oracle.rel_frobenius(np32(tail), np32(plain)) <= 1e-5
    rows = np.r_[0:4, M - 260:M - 250, M - 4:M]
    want = oracle.gemm_kseq(np.ascontiguousarray(np32(a)[rows]), np32(b), np32(c0)[rows])
    assert oracle.rel_frobenius(np32(tail)[rows], want) <= 1e-5
    bf = contract("(i,k),(k,j)->(i,j)", a, b, schedule=dict(tile, splits=-3))
    assert oracle.rel_frobenius(np32(bf), np32(plain) - np32(c0)) <= BF16_TOL
    again = contract("(i,k),(k,j)->(i,j)", a, b, schedule=dict(tile, splits=-3))
    assert torch.equal(bf, again)   # deterministic whatever the arrival order


@pytest.mark.parametrize("M,N,K,bn", [(512, 1024, 512, 256), (768, 1280, 640, 256),
                                      (1024, 2560, 8192, 512), (256, 768, 192, 256)])
@pytest.mark.parametrize("a_mn,b_mn", [(False, True), (True, False), (True, True), (False, False)])
def test_cluster_n2_a_multicast_bit_equal(dev, M, N, K, bn, a_mn, b_mn):
    """Two CTA pairs per cluster sharing A by TMA multicast (schedule
    cluster_n=2) compute exactly what one pair computes (same MMA order):
    bit-equal, any operand majorness, odd tile counts along N (the second
    pair's tile falls outside N), f32 out and c0."""
    g = torch.Generator(device=dev).manual_seed(M + N + K)
    a = torch.randn(M, K, device=dev, generator=g).bfloat16()
    b = torch.randn(K, N, device=dev, generator=g).bfloat16()
    a_in = a.t().contiguous().t() if a_mn else a
    b_in = b if b_mn else b.t().contiguous().t()
    for out_dtype, c0 in ((torch.bfloat16, None), (torch.float32, torch.randn(M, N, device=dev))):
        base = contract("(i,k),(k,j)->(i,j)", a_in, b_in, out_dtype=out_dtype, c0=c0,
                        schedule={"tile_n": bn, "cta_group": 2, "cluster_n": 1, "no_splitk": 1})
        y = contract("(i,k),(k,j)->(i,j)", a_in, b_in, out_dtype=out_dtype, c0=c0,
                     schedule={"tile_n": bn, "cta_group": 2, "cluster_n": 2, "no_splitk": 1})
        assert torch.equal(y, base)
    want = a.double() @ b.double()
    assert float((base.double() - want - c0.double()).norm() / want.norm()) < 1e-5


def test_cluster_n2_batched(dev):
    a = torch.randn(6, 384, 512, device=dev).half()
    b = torch.randn(6, 512, 640, device=dev).half()
    sc = {"tile_n": 256, "cta_group": 2}
    base = contract("(b,i,k),(b,k,j)->(b,i,j)", a, b, schedule=dict(sc, cluster_n=1))
    y = contract("(b,i,k),(b,k,j)->(b,i,j)", a, b, schedule=dict(sc, cluster_n=2))
    assert torch.equal(y, base)


def test_auto_cluster_choice_is_bit_equal(dev):
    """4096^3: the automatic choice (A-multicast clusters when they need no
    more waves) gives exactly the single-pair result."""
    a = torch.randn(4096, 4096, device=dev).bfloat16()
    b = torch.randn(4096, 4096, device=dev).bfloat16()
    auto = contract("(i,k),(k,j)->(i,j)", a, b)
    one = contract("(i,k),(k,j)->(i,j)", a, b, schedule={"cluster_n": 1})
    assert torch.equal(auto, one)


def test_tail_split_batched_and_f16(dev):
    """Tail split with a batch index and fp16 in/out: matches the unsplit
    kernel to f32 noise and is deterministic."""
    a = torch.randn(3, 1280, 2048, device=dev).half()
    b = torch.randn(3, 2048, 1536, device=dev).half()
    spec = "(b,i,k),(b,k,j)->(b,i,j)"
    plain = contract(spec, a, b, out_dtype=torch.float32, schedule={"splits": 1})
    for sp in (-2, -3):
        executor.reset_launch_log()
        tail = contract(spec, a, b, out_dtype=torch.float32, schedule={"splits": sp})
        assert executor.launch_log() == ["tcgen05-tailsplit"], executor.launch_log()
        assert float((tail - plain).norm() / plain.norm()) <= 1e-6
        again = contract(spec, a, b, out_dtype=torch.float32, schedule={"splits": sp})
        assert torch.equal(tail, again)


def test_cluster_n2_with_uniform_splitk(dev):
    """A-multicast clusters combined with uniform split-K slices."""
    a = torch.randn(512, 65536, device=dev).bfloat16()
    b = torch.randn(65536, 1024, device=dev).bfloat16()
    sc = {"tile_n": 256, "cta_group": 2, "splits": 4}
    base = contract("(i,k),(k,j)->(i,j)", a, b, out_dtype=torch.float32,
                    schedule=dict(sc, cluster_n=1))
    executor.reset_launch_log()
    y = contract("(i,k),(k,j)->(i,j)", a, b, out_dtype=torch.float32, schedule=dict(sc, cluster_n=2))
    assert executor.launch_log() == ["tcgen05-splitk"]
    assert torch.equal(y, base)


def test_gemm_fuzz_shapes_layouts_schedules(dev):
    """Randomised shapes (ragged M/N/K, batch), operand majorness, output
    dtype, c0 and schedules (tile, CTA pair, A-multicast clusters, split-K,
    tail split) against an f64 product: relF <= 1e-2, and no device fault."""
    import random
    r = random.Random(4711)
    scheds = [None, {"tile_n": 128, "cta_group": 1}, {"tile_n": 256, "cta_group": 2},
              {"tile_n": 512, "cta_group": 2}, {"cta_group": 2, "tile_n": 256, "cluster_n": 2},
              {"splits": 3}, {"splits": -2}, {"tile_n": 64, "cta_group": 1, "raster": -4}]
    for it in range(200):
        bt = r.choice([1, 1, 1, 3])
        M = r.randint(1, 1500)
        N = 8 * r.randint(1, 300) if r.random() < 0.8 else r.randint(1, 2400)
        K = r.choice([8, 64, 200, 1000, 4104]) if r.random() < 0.8 else r.randint(1, 5000)
        dt = r.choice([torch.bfloat16, torch.float16])
        a = torch.randn(bt, M, K, device=dev).to(dt)
        b = torch.randn(bt, K, N, device=dev).to(dt)
        if r.random() < 0.3:
            a = a.transpose(1, 2).contiguous().transpose(1, 2)
        if r.random() < 0.3:
            b = b.transpose(1, 2).contiguous().transpose(1, 2)
        out_dt = r.choice([dt, torch.float32])
        c0 = torch.randn(bt, M, N, device=dev).to(out_dt) if r.random() < 0.3 else None
        sc = r.choice(scheds)
        y = contract("(b,i,k),(b,k,j)->(b,i,j)", a, b, c0=c0, out_dtype=out_dt, schedule=sc)
        torch.cuda.synchronize()
        want = a.double() @ b.double() + (c0.double() if c0 is not None else 0)
        err = float((y.double() - want).norm() / want.norm())
        assert err <= 1e-2, (it, bt, M, N, K, dt, out_dt, sc, err)


@pytest.mark.parametrize("M,N,K,with_c0", [(2048, 1001, 999, False), (1500, 4095, 2049, True),
                                           (3000, 640, 1003, True)])
def test_unaligned_16bit_gemm_padded_onto_tensor_cores(dev, M, N, K, with_c0):
    """16-bit GEMMs with odd K / N (not TMA-legal) are zero-padded onto the
    tensor cores instead of the CUDA-core fallback: tolerance vs f64, and
    the launch log shows tcgen05."""
    a = torch.randn(M, K, device=dev).bfloat16()
    b = torch.randn(K, N, device=dev).bfloat16()
    c0 = torch.randn(M, N, device=dev).bfloat16() if with_c0 else None
    executor.reset_launch_log()
    y = contract("(i,k),(k,j)->(i,j)", a, b, c0=c0)
    assert any(k.startswith("tcgen05") for k in executor.launch_log()), executor.launch_log()
    want = a.double() @ b.double() + (c0.double() if c0 is not None else 0)
    assert float((y.double() - want).norm() / want.norm()) <= 1e-2
    # strided output view
    big = torch.zeros(M, N + 5, device=dev, dtype=torch.bfloat16)
    contract("(i,k),(k,j)->(i,j)", a, b, c0=c0, out=big[:, 2:N + 2])
    assert torch.equal(big[:, 2:N + 2], y)


def test_tc_and_tf32_modes_pad_odd_shapes(dev):
    """The tensor-core-only modes pad odd shapes instead of failing."""
    a = torch.randn(300, 203, device=dev)
    b = torch.randn(203, 101, device=dev)
    y = contract("(i,k),(k,j)->(i,j)", a, b, mode="tf32")
    want = a.double() @ b.double()
    assert float((y.double() - want).norm() / want.norm()) <= 5e-3
    ah, bh = a.bfloat16(), b.bfloat16()
    executor.reset_launch_log()
    y = contract("(i,k),(k,j)->(i,j)", ah, bh, mode="tc")
    assert any(k.startswith("tcgen05") for k in executor.launch_log())
    assert float((y.double() - ah.double() @ bh.double()).norm() / want.norm()) <= 1e-2


@pytest.mark.parametrize("bt,m,n,k", [(4096, 8, 8, 8), (1024, 16, 16, 16), (512, 32, 32, 32),
                                      (2048, 4, 4, 64)])
def test_small_batched_gemms(dev, bt, m, n, k):
    """Many tiny matrices go to the loop nest (plan 'small batched GEMM'):
    f32 bit-identical to the reference order, bf16 within the tolerance."""
    a = rnd((bt, m, k), 91, dev)
    b = rnd((bt, k, n), 92, dev)
    got = contract("(b,i,k),(b,k,j)->(b,i,j)", a, b).cpu().numpy()
    A, B = np32(a), np32(b)
    for i in (0, bt // 2, bt - 1):
        assert np.array_equal(got[i], oracle.gemm_kseq(A[i], B[i])), i
    ah, bh = a.bfloat16(), b.bfloat16()
    g16 = contract("(b,i,k),(b,k,j)->(b,i,j)", ah, bh).float().cpu().numpy()
    want = np.einsum("bik,bkj->bij", np32(ah).astype(np.float64), np32(bh).astype(np.float64))
    assert oracle.rel_frobenius(g16, want) <= BF16_TOL


@pytest.mark.parametrize("M,N,K", [(4096, 8, 64), (8, 4096, 64), (3000, 5, 33), (6, 2000, 300)])
def test_skinny_exact_gemms(dev, M, N, K):
    """Exact f32 GEMMs with at most 8 rows or columns run on the loop nest
    (plan 'skinny exact GEMM'): bit-identical to the reference order."""
    a, b = rnd((M, K), 93, dev), rnd((K, N), 94, dev)
    got = contract("(i,k),(k,j)->(i,j)", a, b).cpu().numpy()
    assert np.array_equal(got, oracle.gemm_kseq(np32(a), np32(b)))

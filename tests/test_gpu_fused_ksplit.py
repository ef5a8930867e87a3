"""K-split GEMM fused with the reduce-scatter (bgx_contract_reduce_scatter,
shard.FusedKSplit / emulate_fused_ksplit).  Multi-rank runs are emulated on
one GPU exactly as bgx.h describes (one launch per rank in rank order, no
launch waits for another); tolerance relF <= 1e-2 for bf16/fp16 against an
f64 product of the same inputs, and bitwise-deterministic results."""

import os
import socket

import pytest
import torch

from paper_2503_04771_b200 import _lib, executor, shard

pytestmark = pytest.mark.gpu
MM = "(i,k),(k,j)->(i,j)"


def _relf(got, want):
    return float((got.double() - want).norm() / want.norm())


def _slabs(a, b, world, ks=None):
    K = a.shape[1]
    bounds = ks or [shard.k_range(K, world, r) for r in range(world)]
    return [a[:, lo:hi] for lo, hi in bounds], [b[lo:hi] for lo, hi in bounds]


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("M,N,K", [(1024, 1024, 16384), (4096, 512, 8192), (1000, 1000, 4096),
                                   (384, 256, 8192), (200, 512, 4096)])
def test_emulated_reduce_scatter_matches(dev, world, M, N, K):
    g = torch.Generator(device=dev).manual_seed(M + N + world)
    a = torch.randn(M, K, device=dev, generator=g).bfloat16()
    b = torch.randn(K, N, device=dev, generator=g).bfloat16()
    want = a.double() @ b.double()
    A, B = _slabs(a, b, world)
    executor.reset_launch_log()
    out = shard.emulate_fused_ksplit(MM, A, B)
    # default (deferred) mode: world delivering GEMMs, then each owner's reduce
    assert executor.launch_log() == ["tcgen05-rs"] * world + ["rs-reduce"] * world
    assert out.shape == (M, N) and out.dtype == torch.bfloat16
    assert _relf(out, want) < 1e-2
    again = shard.emulate_fused_ksplit(MM, A, B)
    assert torch.equal(out.view(torch.int16), again.view(torch.int16))   # deterministic


@pytest.mark.parametrize("out_dtype", [torch.float32, torch.float16])
def test_emulated_with_c0_ragged_k(dev, out_dtype):
    M, N = 768, 640
    ks = [(0, 3072), (3072, 4160), (4160, 9216)]          # uneven K slabs
    a = torch.randn(M, 9216, device=dev).half()
    b = torch.randn(9216, N, device=dev).half()
    c0 = torch.randn(M, N, device=dev).to(out_dtype)
    A, B = _slabs(a, b, 3, ks)
    out = shard.emulate_fused_ksplit(MM, A, B, c0=c0, out_dtype=out_dtype)
    want = a.double() @ b.double() + c0.double()
    assert out.dtype == out_dtype
    assert _relf(out, want) < (1e-5 if out_dtype == torch.float32 else 1e-2)


def test_plan_tiles_and_ownership(dev):
    a = torch.empty(1024, 2048, device=dev, dtype=torch.bfloat16)
    b = torch.empty(2048, 1024, device=dev, dtype=torch.bfloat16)
    pl = shard.rs_plan(MM, a, b, 8)
    assert (pl.cta_group, pl.rows_per_owner) == (2, 128)
    pl2 = shard.rs_plan(MM, torch.empty(4096, 2048, device=dev, dtype=torch.bfloat16), b, 2)
    assert (pl2.cta_group, pl2.tile_n, pl2.rows_per_owner) == (2, 256, 2048)
    assert pl.mode == _lib.RS_DEFERRED and pl.ws_bytes == 0
    assert pl.local_splits >= 1 and pl.slot_bytes == 8 * pl.local_splits * 128 * 1024 * 4


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("splits", [None, 1, 3])
def test_deferred_and_in_kernel_modes_bit_identical(dev, world, splits):
    """Both reduction placements sum the same partials in the same order
    (slices inside a rank, ranks in rank order, then c0): identical bits,
    with ragged K slabs, c0 and a forced local split."""
    M, N, K = 640, 384, 6144 + 64 * world
    g = torch.Generator(device=dev).manual_seed(world * 7 + (splits or 0))
    a = torch.randn(M, K, device=dev, generator=g).bfloat16()
    b = torch.randn(K, N, device=dev, generator=g).bfloat16()
    c0 = torch.randn(M, N, device=dev, generator=g).bfloat16()
    ks = {1: [(0, K)], 2: [(0, 2048), (2048, K)],
          3: [(0, 1024), (1024, 4096), (4096, K)]}.get(world)     # ragged K slabs
    A, B = _slabs(a, b, world, ks)
    outs = [shard.emulate_fused_ksplit(MM, A, B, c0=c0, mode=m, local_splits=splits)
            for m in (_lib.RS_IN_KERNEL, _lib.RS_DEFERRED)]
    assert torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16))
    assert _relf(outs[1], a.double() @ b.double() + c0.double()) < 1e-2


def test_deferred_rejects_split_beyond_k_blocks(dev):
    a = torch.randn(256, 128, device=dev).bfloat16()     # 2 k-blocks
    b = torch.randn(128, 256, device=dev).bfloat16()
    d, _ = shard._rs_desc(MM, a, b, torch.bfloat16)
    pl = shard.rs_plan(MM, a, b, 1)
    shard._finish_plan(pl, 256, 256, 4, _lib.RS_DEFERRED)
    rs = _lib.BgxReduceScatter()
    buf = torch.zeros(pl.slot_bytes + 4096, dtype=torch.uint8, device=dev)
    rs.plan, rs.slots[0], rs.counters[0], rs.out[0] = pl, buf.data_ptr(), buf.data_ptr(), buf.data_ptr()
    lib = _lib.load()
    assert lib.bgx_contract_reduce_scatter(d, rs, None) == _lib.ERR_INVALID
    assert b"k-blocks" in lib.bgx_last_error()


def test_transposed_operands(dev):
    """MN-major A (k,i) and K-major B (j,k) through the same fused kernel."""
    M, N, K = 512, 768, 8192
    at = torch.randn(K, M, device=dev).bfloat16()
    bt = torch.randn(N, K, device=dev).bfloat16()
    spec = "(k,i),(j,k)->(i,j)"
    A = [at[lo:hi] for lo, hi in (shard.k_range(K, 2, r) for r in range(2))]
    B = [bt[:, lo:hi] for lo, hi in (shard.k_range(K, 2, r) for r in range(2))]
    out = shard.emulate_fused_ksplit(spec, A, B)
    assert _relf(out, at.double().T @ bt.double().T) < 1e-2


def test_fused_single_rank_object(dev):
    a = torch.randn(512, 32768, device=dev).bfloat16()
    b = torch.randn(32768, 256, device=dev).bfloat16()
    f = shard.FusedKSplit(MM, a, b)
    y = f(a, b)
    assert _relf(y, a.double() @ b.double()) < 1e-2
    y2 = f(a, b).clone()
    assert torch.equal(y.view(torch.int16), y2.view(torch.int16))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_fused_symmetric_memory_world1(dev):
    """The real multi-GPU code path (symmetric-memory rendezvous, device
    barriers, peer pointers from the handle) at world size 1."""
    import torch.distributed as dist
    if dist.is_initialized():
        pytest.skip("process group already initialised")
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        a = torch.randn(256, 16384, device=dev).bfloat16()
        b = torch.randn(16384, 512, device=dev).bfloat16()
        c0 = torch.randn(256, 512, device=dev).bfloat16()
        f = shard.FusedKSplit(MM, a, b, with_c0=True)
        assert f.hdl is not None and f.world == 1
        y = f(a, b, c0=c0)
        assert _relf(y, a.double() @ b.double() + c0.double()) < 1e-2
    finally:
        dist.destroy_process_group()


def test_ksplit_contract_fused_flag_single_rank(dev):
    a = torch.randn(384, 8192, device=dev).bfloat16()
    b = torch.randn(8192, 256, device=dev).bfloat16()
    y = shard.ksplit_contract(MM, a, b, scatter=True, fused=True)
    assert _relf(y, a.double() @ b.double()) < 1e-2
    y2 = shard.ksplit_contract(MM, a, b, scatter=True, fused=True)   # cached object
    assert torch.equal(y.view(torch.int16), y2.view(torch.int16))
    with pytest.raises(ValueError, match="scatter=True"):
        shard.ksplit_contract(MM, a, b, fused=True)


def test_ksplit_contract_fused_result_not_aliased(dev):
    """the returned slab must survive the next call with the same
    shapes (it used to be a view into the plan's symmetric buffer), caller
    `out=` is honoured, and the plan cache is bounded (evicted plans release
    their buffers)."""
    a = torch.randn(256, 4096, device=dev).bfloat16()
    b = torch.randn(4096, 256, device=dev).bfloat16()
    y1 = shard.ksplit_contract(MM, a, b, scatter=True, fused=True)
    keep = y1.clone()
    shard.ksplit_contract(MM, 2 * a, b, scatter=True, fused=True)
    assert torch.equal(y1, keep)
    out = torch.empty_like(y1)
    r = shard.ksplit_contract(MM, a, b, scatter=True, fused=True, out=out)
    assert r is out and torch.equal(out, keep)
    plans = []
    for n in range(shard.FUSED_CACHE_LIMIT + 2):
        bn = torch.randn(4096, 128 + 64 * n, device=dev).bfloat16()
        shard.ksplit_contract(MM, a, bn, scatter=True, fused=True)
        plans.append(next(reversed(shard._FUSED_CACHE.values())))
    assert len(shard._FUSED_CACHE) <= shard.FUSED_CACHE_LIMIT
    assert plans[0].buf is None            # evicted: buffer released
    with pytest.raises(RuntimeError, match="after close"):
        plans[0](a, torch.randn(4096, 128, device=dev).bfloat16())


@pytest.mark.parametrize("M,world", [(300, 4), (130, 2), (129, 8), (640, 3)])
def test_emulated_ragged_owners(dev, M, world):
    """Owners with partial or no rows (rows_per_owner rounded to 128)."""
    N, K = 384, 2048 * world
    a = torch.randn(M, K, device=dev).bfloat16()
    b = torch.randn(K, N, device=dev).bfloat16()
    A, B = _slabs(a, b, world)
    out = shard.emulate_fused_ksplit(MM, A, B, out_dtype=torch.float32)
    assert out.shape == (M, N)
    assert _relf(out, a.double() @ b.double()) < 1e-5


def test_fused_reduce_scatter_fuzz(dev):
    """Random world sizes, ragged M, N, uneven K slabs, c0 and output dtype."""
    import random
    r = random.Random(99)
    for it in range(25):
        world = r.randint(1, 8)
        M = r.randint(1, 1200)
        N = 8 * r.randint(1, 160)
        ks = sorted(r.sample(range(8, 8 * 900, 8), world - 1)) if world > 1 else []
        bounds = list(zip([0] + ks, ks + [8 * 900]))
        a = torch.randn(M, 8 * 900, device=dev).bfloat16()
        b = torch.randn(8 * 900, N, device=dev).bfloat16()
        out_dt = r.choice([torch.bfloat16, torch.float32])
        c0 = torch.randn(M, N, device=dev).to(out_dt) if r.random() < 0.5 else None
        A, B = _slabs(a, b, world, bounds)
        y = shard.emulate_fused_ksplit(MM, A, B, c0=c0, out_dtype=out_dt)
        torch.cuda.synchronize()
        want = a.double() @ b.double() + (c0.double() if c0 is not None else 0)
        assert _relf(y, want) < 1e-2, (it, world, M, N, out_dt)


def test_ksplit_demo_size_world8(dev):
    """SURVEY §8e K-split demo at full size (1024 x 1024, K = 2^21 over 8
    emulated ranks): f64 row samples, exact scaling by 2, both reduction
    placements bit-identical."""
    import numpy as np

    import oracle
    M = N = 1024
    K = 1 << 21
    g = torch.Generator(device=dev).manual_seed(21)
    a = torch.randn(M, K, device=dev, generator=g).bfloat16()
    b = torch.randn(K, N, device=dev, generator=g).bfloat16()
    A, B = _slabs(a, b, 8)
    out = shard.emulate_fused_ksplit(MM, A, B)
    rows = np.random.default_rng(4).choice(M, 4, replace=False)
    ar = a[torch.as_tensor(rows, device=dev)].double()
    want = (ar @ b.double()).cpu().numpy()
    got = out[torch.as_tensor(rows, device=dev)].float().cpu().numpy()
    assert oracle.rel_frobenius(got, want) <= 1e-2
    twice = shard.emulate_fused_ksplit(MM, [x * 2 for x in A], B)
    assert torch.equal(twice, out * 2)
    ink = shard.emulate_fused_ksplit(MM, A, B, mode=_lib.RS_IN_KERNEL)
    assert torch.equal(ink.view(torch.int16), out.view(torch.int16))

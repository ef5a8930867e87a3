"""Multi-process host logic on CPU (gloo, world_size 2): the M-shard row
partition and the K-split reduction (reduce-scatter / all-reduce) that the
B200 path runs over NCCL.  The local per-rank contraction is replaced here by
a torch CPU matmul stand-in — the kernels themselves are covered by the gpu
tests; this checks the data-movement logic around them."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_04771_b200 import shard


def test_row_range_partitions():
    for total in (1, 127, 128, 1000, 32768, 32769):
        for world in (1, 2, 3, 4, 8):
            spans = [shard.row_range(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b
            for a, b in spans[:-1]:
                assert a % 128 == 0 or a == total


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cpu_cast(src, out, c0):
    v = src if c0 is None else src + c0.float()
    out.copy_(v.to(out.dtype))
    return out


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(0)
        M, N, K = 64, 48, 96
        A = torch.randn(M, K, generator=g)
        B = torch.randn(K, N, generator=g)
        C0 = torch.randn(M, N, generator=g)
        full = A @ B
        k0, k1 = shard.k_range(K, world, rank, align=16)
        partial = A[:, k0:k1] @ B[k0:k1]                 # stand-in for the tcgen05 partial
        red = shard.ksplit_reduce(partial.clone(), group=None)
        ok_ar = torch.allclose(red, full, rtol=1e-5, atol=1e-4)
        rs = shard.ksplit_reduce(partial.clone(), c0=C0, out_dtype=torch.float32, scatter=True,
                                 cast=_cpu_cast)
        rows = M // world
        ok_rs = torch.allclose(rs, (full + C0)[rank * rows:(rank + 1) * rows], rtol=1e-5, atol=1e-4)
        bf = shard.ksplit_reduce(partial.clone(), out_dtype=torch.bfloat16, cast=_cpu_cast)
        ok_bf = bf.dtype == torch.bfloat16 and torch.allclose(bf.float(), full, rtol=1e-2, atol=1e-1)
        # M-shard: no collective on the data path; gather only to check
        r0, r1 = shard.row_range(M, world, rank, align=16)
        mine = A[r0:r1] @ B
        parts = [torch.empty(0)] * world
        dist.all_gather_object(parts, (r0, r1, mine))
        stitched = torch.cat([p[2] for p in sorted(parts, key=lambda t: t[0])])
        ok_m = torch.allclose(stitched, full, rtol=1e-5, atol=1e-4)
        q.put((rank, ok_ar, ok_rs, ok_bf, ok_m))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_ksplit_and_mshard_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    results = sorted(q.get() for _ in range(world))
    for rank, *oks in results:
        assert all(oks), (rank, oks)


@pytest.mark.parametrize("M,world", [(1, 1), (300, 4), (1024, 8), (129, 8), (4096, 3), (100000, 7)])
def test_fused_rs_row_ownership_partitions_rows(M, world):
    """The fused reduce-scatter's ownership (rows_per_owner = ceil(M/world)
    rounded up to 128, as bgx_contract_rs_plan computes it) covers every
    output row exactly once, in rank order."""
    from paper_2503_04771_b200 import shard
    rpo = -(-(-(-M // world)) // 128) * 128
    spans = [shard.owned_rows(M, rpo, r) for r in range(world)]
    covered = [i for lo, hi in spans for i in range(lo, hi)]
    assert covered == list(range(M))
    assert all(lo <= hi for lo, hi in spans)


_SHARD_SPECS = [("(i,k),(k,j)->(i,j)", [(300, 40), (40, 24)]),
                ("(k,i),(k,j)->(i,j)", [(40, 300), (40, 24)]),
                ("(k,j),(i,k)->(i,j)", [(40, 24), (300, 40)]),
                ("(i,j)->(j,i)", [(50, 333)]),
                ("(i,j,k)->(k,j,i)", [(7, 9, 260)]),
                ("(i,k),(k,j),(j,l)->(i,l)", [(257, 16), (16, 8), (8, 12)])]


def _torch_einsum(spec, ops):
    """CPU stand-in for the per-rank contraction (bracket spec -> torch.einsum)."""
    from paper_2503_04771_b200.einsum import EinsumSpec, parse_einsum
    sp = spec if isinstance(spec, EinsumSpec) else parse_einsum(spec)
    letters = {ax: chr(97 + n) for n, ax in enumerate(sp.axes)}
    eq = ",".join("".join(letters[a] for a in t) for t in sp.inputs)
    return torch.einsum(eq + "->" + "".join(letters[a] for a in sp.output), *ops)


def _shard_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        oks = []
        for n, (spec, shapes) in enumerate(_SHARD_SPECS):
            g = torch.Generator().manual_seed(n)
            ops = [torch.randn(s, generator=g, dtype=torch.float64) for s in shapes]
            lo, hi, local = shard.shard_operands(spec, ops, world, rank, align=16)
            mine = _torch_einsum(spec, local)
            parts = [None] * world
            dist.all_gather_object(parts, (lo, hi, mine))
            stitched = torch.cat([p[2] for p in sorted(parts, key=lambda t: t[0])])
            oks.append(torch.allclose(stitched, _torch_einsum(spec, ops), rtol=1e-12, atol=1e-12))
        q.put((rank, *oks))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_shard_operands_gloo(world):
    """§8e M-shard for any leading output index (operand 0 or 1, strided
    slabs, permutations, the chain): stitched per-rank slabs equal the whole."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    for rank, *oks in sorted(q.get() for _ in range(world)):
        assert all(oks), (rank, oks)


def test_lead_slabs_views():
    """lead_slabs narrows exactly the operands carrying the output's leading
    index, along that index, without copying."""
    a, b = torch.randn(40, 300), torch.randn(40, 24)
    sa, sb = shard.lead_slabs("(k,i),(k,j)->(i,j)", [a, b], 100, 164)
    assert sa.shape == (40, 64) and sa.data_ptr() == a[:, 100:].data_ptr() and sb is b
    with pytest.raises(ValueError, match="rank-0"):
        shard.lead_slabs("(i),(i)->()", [a[0], a[1]], 0, 1)


def _sharded_contract_worker(rank, world, port, q):
    """shard.sharded_contract's host logic (rank/world from the process group,
    the slab views, the c0 slab) with the per-rank contraction stood in by
    torch.einsum on CPU (the CUDA path is tests/test_gpu_sharded.py)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def fake_contract(spec, *ops, c0=None, **kw):
            out = _torch_einsum(spec, ops)
            return out if c0 is None else out + c0
        shard.contract = fake_contract
        oks = []
        for n, (spec, shapes) in enumerate(_SHARD_SPECS):
            g = torch.Generator().manual_seed(n)
            ops = [torch.randn(s, generator=g, dtype=torch.float64) for s in shapes]
            full = _torch_einsum(spec, ops)
            c0 = torch.randn(full.shape, generator=g, dtype=torch.float64)
            lo, hi, mine = shard.sharded_contract(spec, *ops, c0=c0, align=16)
            parts = [None] * world
            dist.all_gather_object(parts, (lo, hi, mine))
            stitched = torch.cat([p[2] for p in sorted(parts, key=lambda t: t[0])])
            oks.append(torch.allclose(stitched, full + c0, rtol=1e-12, atol=1e-12))
        q.put((rank, *oks))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_contract_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_contract_worker, args=(r, world, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    for rank, *oks in sorted(q.get() for _ in range(world)):
        assert all(oks), (rank, oks)

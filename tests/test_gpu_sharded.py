"""shard.sharded_contract on the B200: two ranks (gloo process group, both on
cuda:0 — their kernels are independent, no rank waits on another) each
contract their output row slab from replicated operands; the stitched slabs
equal the single-device result bit for bit."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

SPECS = [("(i,k),(k,j)->(i,j)", [(1024, 512), (512, 384)], torch.bfloat16),
         ("(i,k),(k,j),(j,l)->(i,l)", [(768, 256), (256, 256), (256, 128)], torch.bfloat16),
         ("(b,i,k),(b,k,j)->(b,i,j)", [(6, 256, 128), (6, 128, 256)], torch.bfloat16),
         ("(i,j)->(j,i)", [(512, 1000)], torch.float32),
         ("(i,k),(k,j)->(i,j)", [(300, 64), (64, 80)], torch.float32)]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2503_04771_b200 import contract, shard
        dev = torch.device("cuda", 0)
        res = []
        for n, (spec, shapes, dt) in enumerate(SPECS):
            g = torch.Generator(device=dev).manual_seed(n)
            ops = [torch.randn(s, generator=g, device=dev).to(dt) for s in shapes]
            lo, hi, mine = shard.sharded_contract(spec, *ops)
            parts = [None] * world
            dist.all_gather_object(parts, (lo, hi, mine.cpu()))
            stitched = torch.cat([p[2] for p in sorted(parts, key=lambda t: t[0])])
            res.append(bool(torch.equal(stitched, contract(spec, *ops).cpu())))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_sharded_contract_two_ranks(dev):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    for rank, res in sorted(q.get() for _ in range(2)):
        assert all(res), (rank, res)

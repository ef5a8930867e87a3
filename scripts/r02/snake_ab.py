"""A/B of the K-direction snake (debug bit 8192: every other persistent
iteration walks K backwards, so a wave starts on the K-panels the previous
wave touched last) on GEMM shapes: interleaved blocks of back-to-back
launches, sustained per-launch time.  python scripts/r02/snake_ab.py SHAPE..."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts/r02")
from paper_2503_04771_b200 import _lib  # noqa: E402
from probe_drain import SHAPES  # noqa: E402

lib = _lib.load()
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream().cuda_stream
for shape in sys.argv[1:] or ["chain"]:
    bt, M, N, K = SHAPES[shape]
    a = torch.randn(bt, M, K, device=dev).bfloat16()
    b = torch.randn(bt, K, N, device=dev).bfloat16()
    outs = {}
    descs = {}
    for dbg in (0, 8192):
        out = torch.empty(bt, M, N, device=dev, dtype=torch.bfloat16)
        d = _lib.BgxContractDesc()
        d.batch, d.M, d.N, d.K = bt, M, N, K
        d.a, d.b, d.out = a.data_ptr(), b.data_ptr(), out.data_ptr()
        d.a_stride[:] = [M * K, K, 1]
        d.b_stride[:] = [K * N, N, 1]
        d.o_stride[:] = [M * N, N, 1]
        d.in_dtype = d.out_dtype = _lib.BF16
        d.mode = _lib.MODE_TC
        d.sched.reserved[0] = dbg
        descs[dbg], outs[dbg] = d, out
    flop = 2 * bt * M * N * K
    n = max(4, int(0.15e15 / flop * 0 + 200e-3 / (flop / 1.4e15)))   # ~200 ms blocks
    res = {0: [], 8192: []}
    for _ in range(2):
        for d in descs.values():
            _lib.check(lib.bgx_contract(d, st), "w")
    torch.cuda.synchronize()
    for rnd in range(6):
        for dbg in ((0, 8192) if rnd % 2 == 0 else (8192, 0)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(n):
                _lib.check(lib.bgx_contract(descs[dbg], st), "r")
            e1.record()
            torch.cuda.synchronize()
            res[dbg].append(e0.elapsed_time(e1) / n)
    rel = ((outs[0].float() - outs[8192].float()).norm() / outs[0].float().norm()).item()
    for dbg in (0, 8192):
        ms = statistics.median(res[dbg])
        print(f"{shape:7s} {'snake' if dbg else 'plain':6s} {ms*1e3:8.1f} us  {flop/ms/1e9:7.1f} TFLOP/s"
              f"  blocks={[round(x*1e3,1) for x in res[dbg]]}", flush=True)
    print(f"{shape:7s} relF(snake vs plain) = {rel:.2e}", flush=True)

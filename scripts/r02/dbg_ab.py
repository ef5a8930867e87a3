"""A/B of two schedule debug settings (default: 0 vs 16384 = direct
epilogue off) on GEMM shapes: interleaved blocks of back-to-back launches
(~200 ms each, power-capped steady state) plus short bursts after 0.5 s idle.
python scripts/r02/dbg_ab.py [--bits A,B] SHAPE..."""
import time
import statistics
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts/r02")
from paper_2503_04771_b200 import _lib  # noqa: E402
from probe_drain import SHAPES  # noqa: E402

args = sys.argv[1:]
BITS = ("0", "16384")
if args and args[0] == "--bits":
    BITS = tuple(args[1].split(","))   # "debug" or "debug/cluster_n"
    args = args[2:]
lib = _lib.load()
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream().cuda_stream
for shape in args or ["c3"]:
    bt, M, N, K = SHAPES[shape]
    a = torch.randn(bt, M, K, device=dev).bfloat16()
    b = torch.randn(bt, K, N, device=dev).bfloat16()
    outs = {}
    descs = {}
    for dbg in BITS:
        out = torch.empty(bt, M, N, device=dev, dtype=torch.bfloat16)
        d = _lib.BgxContractDesc()
        d.batch, d.M, d.N, d.K = bt, M, N, K
        d.a, d.b, d.out = a.data_ptr(), b.data_ptr(), out.data_ptr()
        d.a_stride[:] = [M * K, K, 1]
        d.b_stride[:] = [K * N, N, 1]
        d.o_stride[:] = [M * N, N, 1]
        d.in_dtype = d.out_dtype = _lib.BF16
        d.mode = _lib.MODE_TC
        dv, _, cn = dbg.partition("/")
        d.sched.reserved[0] = int(dv)
        d.sched.reserved[1] = int(cn or 0)
        descs[dbg], outs[dbg] = d, out
    flop = 2 * bt * M * N * K
    n = max(4, int(0.15e15 / flop * 0 + 200e-3 / (flop / 1.4e15)))   # ~200 ms blocks
    res = {x: [] for x in BITS}
    burst = {x: [] for x in BITS}
    for _ in range(2):
        for d in descs.values():
            _lib.check(lib.bgx_contract(d, st), "w")
    torch.cuda.synchronize()
    for rnd in range(6):
        for dbg in (BITS if rnd % 2 == 0 else BITS[::-1]):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(n):
                _lib.check(lib.bgx_contract(descs[dbg], st), "r")
            e1.record()
            torch.cuda.synchronize()
            res[dbg].append(e0.elapsed_time(e1) / n)
    for rnd in range(6):
        for dbg in (BITS if rnd % 2 == 0 else BITS[::-1]):
            time.sleep(0.5)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                _lib.check(lib.bgx_contract(descs[dbg], st), "r")
            e1.record()
            torch.cuda.synchronize()
            burst[dbg].append(e0.elapsed_time(e1) / 5)
    same = torch.equal(outs[BITS[0]], outs[BITS[1]])
    for dbg in BITS:
        ms = statistics.median(res[dbg])
        bms = statistics.median(burst[dbg])
        print(f"{shape:7s} debug={dbg:<8s} sustained {ms*1e3:8.1f} us {flop/ms/1e9:7.1f} TFLOP/s | burst "
              f"{bms*1e3:8.1f} us {flop/bms/1e9:7.1f} TFLOP/s  blocks={[round(x*1e3,1) for x in res[dbg]]}",
              flush=True)
    print(f"{shape:7s} outputs bit-identical across settings: {same}", flush=True)

"""Tile / pipeline sweep of the tcgen05 GEMM with direct C-ABI calls (no
Python planning inside the timed region).  Prints one line per config."""
import argparse
import itertools
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="4096x4096x4096,32768x8192x8192")
ap.add_argument("--cg", default="1,2")
ap.add_argument("--bn", default="128,256")
ap.add_argument("--stages", default="0")
ap.add_argument("--raster", default="0")
ap.add_argument("--debug", default="0")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--batch", type=int, default=1)
args = ap.parse_args()
lib = _lib.load()
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream()
flush_buf = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

for shape in args.shapes.split(","):
    M, N, K = (int(x) for x in shape.split("x"))
    Bt = args.batch
    a = torch.randn(Bt, M, K, device=dev).bfloat16()
    b = torch.randn(Bt, K, N, device=dev).bfloat16()
    out = torch.empty(Bt, M, N, device=dev, dtype=torch.bfloat16)
    for cg, bn, st, ra, dbg in itertools.product(*(map(int, v.split(",")) for v in
                                                   (args.cg, args.bn, args.stages, args.raster, args.debug))):
        d = _lib.BgxContractDesc()
        d.batch, d.M, d.N, d.K = Bt, M, N, K
        d.a, d.b, d.out = a.data_ptr(), b.data_ptr(), out.data_ptr()
        d.a_stride[:] = [M * K, K, 1]
        d.b_stride[:] = [K * N, N, 1]
        d.o_stride[:] = [M * N, N, 1]
        d.in_dtype = d.out_dtype = _lib.BF16
        d.mode = _lib.MODE_TC
        d.sched.cta_group, d.sched.tile_n, d.sched.stages, d.sched.raster = cg, bn, st, ra
        d.sched.reserved[0] = dbg
        sp = stream.cuda_stream
        for _ in range(3):
            _lib.check(lib.bgx_contract(d, sp), "warm")
        ts = []
        for _ in range(args.iters):
            flush_buf.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            lib.bgx_contract(d, sp)
            e1.record(stream)
            ts.append((e0, e1))
        torch.cuda.synchronize()
        ms = statistics.median(x.elapsed_time(y) for x, y in ts)
        print(f"{shape} cg={cg} bn={bn} stages={st} raster={ra} debug={dbg}: {ms:.4f} ms "
              f"{2 * Bt * M * N * K / ms / 1e9:.1f} TFLOP/s", flush=True)

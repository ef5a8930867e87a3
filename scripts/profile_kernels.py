"""Short driver for ncu captures: a few launches of each hot kernel at the
BASELINE sizes (run plain first, then under ncu; see B200_PROFILING.md)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200 import contract  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--what", default="gemm4096,chain_gemm,perm8192")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--tile-n", type=int, default=0)
ap.add_argument("--rasters", default="0")
ap.add_argument("--cg", type=int, default=0)
ap.add_argument("--debugs", default="0")
args = ap.parse_args()
dev = torch.device("cuda", 0)
sched = {"tile_n": args.tile_n} if args.tile_n else None
if args.cg:
    sched = dict(sched or {}, cta_group=args.cg)
for what in args.what.split(","):
    if what == "gemm4096":
        a = torch.randn(4096, 4096, device=dev).bfloat16()
        b = torch.randn(4096, 4096, device=dev).bfloat16()
        for _ in range(args.reps):
            contract("(i,k),(k,j)->(i,j)", a, b, schedule=sched)
    elif what == "chain_gemm":
        a = torch.randn(32768, 8192, device=dev).bfloat16()
        b = torch.randn(8192, 8192, device=dev).bfloat16()
        for ra in (int(x) for x in args.rasters.split(",")):
            for dbg in (int(x) for x in args.debugs.split(",")):
                sc = dict(sched or {})
                if ra:
                    sc["raster"] = ra
                if dbg:
                    sc["reserved"] = [dbg, 0, 0]
                for _ in range(args.reps):
                    contract("(i,k),(k,j)->(i,j)", a, b, schedule=sc or None)
    elif what == "batched":
        a = torch.randn(64, 1024, 1024, device=dev).bfloat16()
        b = torch.randn(64, 1024, 1024, device=dev).bfloat16()
        for _ in range(args.reps):
            contract("(b,i,j),(b,j,k)->(b,i,k)", a, b, schedule=sched)
    elif what == "perm8192":
        x = torch.randn(8192, 8192, device=dev)
        for _ in range(args.reps):
            contract("(i,j)->(j,i)", x)
    elif what == "perm3d":
        x = torch.randn(256, 512, 512, device=dev)
        for _ in range(args.reps):
            contract("(i,j,k)->(k,j,i)", x)
torch.cuda.synchronize()
print("done")

"""C3 (64 x 1024^3 bf16) and other shapes: time tile variants with the
kernel's debug probes (reserved[0]: 1 = skip stores, 4 = release the
accumulator without reading TMEM) to locate the per-tile drain cost."""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2503_04771_b200 import _lib  # noqa: E402

SHAPES = {"c3": (64, 1024, 1024, 1024), "c4": (1, 4096, 4096, 4096),
          "r8192": (1, 8192, 8192, 8192), "r16384": (1, 16384, 8192, 8192), "r4096": (1, 4096, 8192, 8192),
          "chain": (1, 32768, 8192, 8192), "k2048": (16, 2048, 2048, 2048)}


def run(shape, variants):
    bt, M, N, K = SHAPES[shape]
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    a = torch.randn(bt, M, K, device=dev).bfloat16()
    b = torch.randn(bt, K, N, device=dev).bfloat16()
    out = torch.empty(bt, M, N, device=dev, dtype=torch.bfloat16)
    st = torch.cuda.current_stream().cuda_stream
    flop = 2 * bt * M * N * K
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ITERS = int(os.environ.get("ITERS", "20")) if M * N * bt < (1 << 28) else 4
    for name, kw in variants:
        d = _lib.BgxContractDesc()
        d.batch, d.M, d.N, d.K = bt, M, N, K
        d.a, d.b, d.out = a.data_ptr(), b.data_ptr(), out.data_ptr()
        d.a_stride[:] = [M * K, K, 1]
        d.b_stride[:] = [K * N, N, 1]
        d.o_stride[:] = [M * N, N, 1]
        d.in_dtype = d.out_dtype = _lib.BF16
        d.mode = _lib.MODE_TC
        for k, v in kw.items():
            if k == "debug":
                d.sched.reserved[0] = v
            elif k == "pf":
                d.sched.reserved[2] = v
            elif k == "cluster_n":
                d.sched.reserved[1] = v
            else:
                setattr(d.sched, k, v)
        fn = lambda: _lib.check(lib.bgx_contract(d, st), "c")  # noqa: E731
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        time.sleep(0.5)          # burst: start from an idle (uncapped) GPU
        ts = []
        for _ in range(ITERS):
            flush.zero_()        # L2 flush between launches (cold operands)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            ts.append((e0, e1))
        torch.cuda.synchronize()
        ms = statistics.median(x.elapsed_time(y) for x, y in ts)
        print(f"{shape:6s} {name:28s} {ms*1e3:9.1f} us {flop/ms/1e9:8.1f} TFLOP/s", flush=True)


VARS = {
    "rows": [("auto", {}), ("t512 r-8", {"tile_n": 512, "cta_group": 2, "raster": -8}),
             ("t512 r-4", {"tile_n": 512, "cta_group": 2, "raster": -4}),
             ("t512 r-16", {"tile_n": 512, "cta_group": 2, "raster": -16}),
             ("t512 r8", {"tile_n": 512, "cta_group": 2, "raster": 8}),
             ("t256", {"tile_n": 256, "cta_group": 2}),
             ("t256 r-8", {"tile_n": 256, "cta_group": 2, "raster": -8})],
    "pf": [("auto", {}), ("auto pf4", {"pf": 4}), ("auto pf8", {"pf": 8}),
           ("auto pf16", {"pf": 16}), ("auto pf32", {"pf": 32}), ("auto again", {})],
    "cn2f": [("t256 quads dyn", {"tile_n": 256, "cta_group": 2, "cluster_n": 2, "debug": 128}),
             ("t256 quads queue-static", {"tile_n": 256, "cta_group": 2, "cluster_n": 2, "debug": 128 + 2048}),
             ("t256 quads static", {"tile_n": 256, "cta_group": 2, "cluster_n": 2, "debug": 128 + 512})],
    "cn2e": [("t256", {"tile_n": 256, "cta_group": 2, "cluster_n": 1}),
             ("t256 quads dyn", {"tile_n": 256, "cta_group": 2, "cluster_n": 2, "debug": 128}),
             ("t256 quads dyn early", {"tile_n": 256, "cta_group": 2, "cluster_n": 2, "debug": 128 + 1024}),
             ("t256 quads static", {"tile_n": 256, "cta_group": 2, "cluster_n": 2, "debug": 128 + 512}),
             ("t256 mixed dyn early", {"tile_n": 256, "cta_group": 2, "cluster_n": 2, "debug": 1024}),
             ("t256 quads dyn noread", {"tile_n": 256, "cta_group": 2, "cluster_n": 2, "debug": 128 + 4}),
             ("t256 quads static noread", {"tile_n": 256, "cta_group": 2, "cluster_n": 2, "debug": 128 + 512 + 4})],
    "cn2q": [("t256", {"tile_n": 256, "cta_group": 2, "cluster_n": 1}),
             ("t256 quads dyn", {"tile_n": 256, "cta_group": 2, "cluster_n": 2, "debug": 128}),
             ("t256 quads static", {"tile_n": 256, "cta_group": 2, "cluster_n": 2, "debug": 128 + 512}),
             ("t256 pairs dyn", {"tile_n": 256, "cta_group": 2, "cluster_n": 2, "debug": 64}),
             ("t256 pairs static", {"tile_n": 256, "cta_group": 2, "cluster_n": 2, "debug": 64 + 512}),
             ("t256 mixed dyn", {"tile_n": 256, "cta_group": 2, "cluster_n": 2})],
    "cn2dbg": [("t256", {"tile_n": 256, "cta_group": 2, "cluster_n": 1}),
               ("t256 cn2", {"tile_n": 256, "cta_group": 2, "cluster_n": 2}),
               ("t256 cn2 pairs-only", {"tile_n": 256, "cta_group": 2, "cluster_n": 2, "debug": 64}),
               ("t256 cn2 quads-only", {"tile_n": 256, "cta_group": 2, "cluster_n": 2, "debug": 128}),
               ("t256 cn2 noread", {"tile_n": 256, "cta_group": 2, "cluster_n": 2, "debug": 4}),
               ("t256 cn2 pairs-only noread", {"tile_n": 256, "cta_group": 2, "cluster_n": 2, "debug": 68})],
    "cn2": [("t256", {"tile_n": 256, "cta_group": 2, "cluster_n": 1}),
            ("t256 cn2", {"tile_n": 256, "cta_group": 2, "cluster_n": 2}),
            ("t512", {"tile_n": 512, "cta_group": 2, "cluster_n": 1}),
            ("t512 cn2", {"tile_n": 512, "cta_group": 2, "cluster_n": 2}),
            ("auto", {})],
    "el": [("t512", {"tile_n": 512, "cta_group": 2}),
           ("t512 e1 l1", {"tile_n": 512, "cta_group": 2, "debug": (1 << 20) | (1 << 16)}),
           ("t512 e2 l2", {"tile_n": 512, "cta_group": 2, "debug": (2 << 20) | (2 << 16)}),
           ("t512 e2 l4", {"tile_n": 512, "cta_group": 2, "debug": (2 << 20) | (4 << 16)}),
           ("t512 e4 l2", {"tile_n": 512, "cta_group": 2, "debug": (4 << 20) | (2 << 16)}),
           ("t512 e1 l4", {"tile_n": 512, "cta_group": 2, "debug": (1 << 20) | (4 << 16)}),
           ("t256", {"tile_n": 256, "cta_group": 2})],
    "late": [("t512 late1", {"tile_n": 512, "cta_group": 2, "debug": 1 << 16}),
             ("t512 late2", {"tile_n": 512, "cta_group": 2, "debug": 2 << 16}),
             ("t512 late3", {"tile_n": 512, "cta_group": 2, "debug": 3 << 16}),
             ("t512 late4", {"tile_n": 512, "cta_group": 2, "debug": 4 << 16})],
    "main": [("auto", {}), ("t256", {"tile_n": 256, "cta_group": 2}),
             ("t512", {"tile_n": 512, "cta_group": 2})],
    "stage": [("t256", {"tile_n": 256, "cta_group": 2}),
              ("t256 stage-only", {"tile_n": 256, "cta_group": 2, "debug": 16}),
              ("t256 store-only", {"tile_n": 256, "cta_group": 2, "debug": 32}),
              ("t256 nostore", {"tile_n": 256, "cta_group": 2, "debug": 1}),
              ("t256 noread", {"tile_n": 256, "cta_group": 2, "debug": 4}),
              ("t512", {"tile_n": 512, "cta_group": 2}),
              ("t512 stage-only", {"tile_n": 512, "cta_group": 2, "debug": 16}),
              ("t512 store-only", {"tile_n": 512, "cta_group": 2, "debug": 32})],
    "depth": [("t256 noread s6", {"tile_n": 256, "cta_group": 2, "debug": 4}),
              ("t256 noread s5", {"tile_n": 256, "cta_group": 2, "debug": 4, "stages": 5}),
              ("t256 noread s4", {"tile_n": 256, "cta_group": 2, "debug": 4, "stages": 4}),
              ("t256 noread s3", {"tile_n": 256, "cta_group": 2, "debug": 4, "stages": 3}),
              ("t512 noread s4", {"tile_n": 512, "cta_group": 2, "debug": 4}),
              ("t512 noread s3", {"tile_n": 512, "cta_group": 2, "debug": 4, "stages": 3}),
              ("t512 noread s2", {"tile_n": 512, "cta_group": 2, "debug": 4, "stages": 2}),
              ("t512 noread r8", {"tile_n": 512, "cta_group": 2, "debug": 4, "raster": 8}),
              ("t512 noread r-2", {"tile_n": 512, "cta_group": 2, "debug": 4, "raster": -2}),
              ("t512 noread r2", {"tile_n": 512, "cta_group": 2, "debug": 4, "raster": 2}),
              ("t256 noread r2", {"tile_n": 256, "cta_group": 2, "debug": 4, "raster": 2}),
              ("t256 noread r-4", {"tile_n": 256, "cta_group": 2, "debug": 4, "raster": -4}),
              ("t128 cg2 noread", {"tile_n": 128, "cta_group": 2, "debug": 4}),
              ("t256 cg1 noread", {"tile_n": 256, "cta_group": 1, "debug": 4})],
}


if __name__ == "__main__":
    if os.environ.get("VARS"):
        for s in sys.argv[1:]:
            run(s, VARS[os.environ["VARS"]])
        sys.exit(0)
    V = [("auto", {}), ("t256", {"tile_n": 256, "cta_group": 2}),
         ("t256 noread", {"tile_n": 256, "cta_group": 2, "debug": 4}),
         ("t256 nostore", {"tile_n": 256, "cta_group": 2, "debug": 1}),
         ("t512", {"tile_n": 512, "cta_group": 2}),
         ("t512 noread", {"tile_n": 512, "cta_group": 2, "debug": 4}),
         ("t512 nostore", {"tile_n": 512, "cta_group": 2, "debug": 1}),
         ("t256 cn2", {"tile_n": 256, "cta_group": 2, "cluster_n": 2}),
         ("t256 cn2 noread", {"tile_n": 256, "cta_group": 2, "cluster_n": 2, "debug": 4})]
    for s in sys.argv[1:] or ["c3"]:
        run(s, V)

"""Interleaved burst/sustained comparison of schedule variants of the same
build (and cuBLAS) on one shape.  Usage:
    python scripts/ab_sched.py SHAPE "raster=8" "raster=-8" "tile_n=512,cta_group=2" ...
(SHAPE as in ab_lib.SHAPES; "" = automatic schedule)."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ab_lib  # noqa: E402
from paper_2503_04771_b200 import _lib  # noqa: E402
from paper_2503_04771_b200.schedule import Schedule  # noqa: E402


def main():
    name = sys.argv[1]
    bt, M, N, K = ab_lib.SHAPES[name]
    lib = _lib.load()
    a = torch.randn(bt, M, K, device=ab_lib.dev).bfloat16()
    b = torch.randn(bt, K, N, device=ab_lib.dev).bfloat16()
    out = torch.empty(bt, M, N, device=ab_lib.dev, dtype=torch.bfloat16)
    impls = {"cublas": lambda: torch.matmul(a, b, out=out)}
    for text in sys.argv[2:]:
        s = Schedule.parse(text)
        dd = _lib.BgxContractDesc()
        dd.batch, dd.M, dd.N, dd.K = bt, M, N, K
        dd.a, dd.b, dd.out = a.data_ptr(), b.data_ptr(), out.data_ptr()
        dd.a_stride[:] = [M * K, K, 1]
        dd.b_stride[:] = [K * N, N, 1]
        dd.o_stride[:] = [M * N, N, 1]
        dd.in_dtype = dd.out_dtype = _lib.BF16
        dd.mode = _lib.MODE_TC
        for k, v in s.to_dict().items():
            if k == "cluster_n":
                dd.sched.reserved[1] = v
            elif k != "splits":
                setattr(dd.sched, k, v)
        st = torch.cuda.current_stream().cuda_stream
        impls[text or "auto"] = (lambda dd=dd: lib.bgx_contract(dd, st))
    flop = 2 * bt * M * N * K
    keys = list(impls)
    for order in (keys, keys[::-1]):
        for impl in order:
            fn = impls[impl]
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            time.sleep(1.0)
            burst = statistics.median(ab_lib.timed(fn, 20))
            sus, mhz = ab_lib.sustained(fn)
            print(json.dumps({"shape": name, "impl": impl, "burst_tflops": round(flop / burst / 1e9, 1),
                              "sustained_tflops": round(flop / sus / 1e9, 1),
                              "sustained_sm_mhz": mhz}), flush=True)


if __name__ == "__main__":
    main()

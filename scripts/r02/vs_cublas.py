"""Our tcgen05 GEMM vs cuBLAS (torch.matmul / torch.bmm) on the BASELINE
shapes, same box, interleaved: burst (after 0.5 s idle, 5 launches) and
sustained (~0.3 s back to back) per-launch device time, plus the in-band SM
clock of each sustained block (bgx_clock_sample: per-SM %clock64 over
%globaltimer), so the per-clock efficiency (TFLOP/s per GHz) can be compared
independently of the power cap.  python scripts/r02/vs_cublas.py"""
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
from bench import inband_clock  # noqa: E402
from paper_2503_04771_b200 import _lib  # noqa: E402

dev = torch.device("cuda", 0)
lib = _lib.load()
st = torch.cuda.current_stream().cuda_stream
nsm = lib.bgx_sm_count()
clk = torch.zeros(2, nsm * 3, dtype=torch.int64, device=dev)

SHAPES = {"C3 64x1024^3": (64, 1024, 1024, 1024), "C4 4096^3": (1, 4096, 4096, 4096),
          "chain GEMM 32768x8192^2": (1, 32768, 8192, 8192), "8192^3": (1, 8192, 8192, 8192)}
if len(sys.argv) > 2:
    SHAPES = {k: v for k, v in SHAPES.items() if k.startswith(sys.argv[2])}


def ours(a, b, o, bt, M, N, K, cn=0, tile_n=0):
    d = _lib.BgxContractDesc()
    d.sched.reserved[1] = cn
    d.sched.tile_n = tile_n
    d.batch, d.M, d.N, d.K = bt, M, N, K
    d.a, d.b, d.out = a.data_ptr(), b.data_ptr(), o.data_ptr()
    d.a_stride[:] = [M * K if bt > 1 else 0, K, 1]
    d.b_stride[:] = [K * N if bt > 1 else 0, N, 1]
    d.o_stride[:] = [M * N if bt > 1 else 0, N, 1]
    d.in_dtype = d.out_dtype = _lib.BF16
    d.mode = _lib.MODE_TC
    return lambda: _lib.check(lib.bgx_contract(d, st), "bgx_contract")


def cublas(a, b, o, bt):
    if bt > 1:
        return lambda: torch.bmm(a, b, out=o)
    return lambda: torch.matmul(a, b, out=o)


def burst(fn):
    time.sleep(0.5)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 5


def sustained(fn, ms_each):
    n = max(5, int(300 / ms_each))
    lib.bgx_clock_sample(clk[0].data_ptr(), st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    lib.bgx_clock_sample(clk[1].data_ptr(), st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n, inband_clock(clk.cpu().numpy())["sm_mhz_inband"]


for name, (bt, M, N, K) in SHAPES.items():
    shp_a = (bt, M, K) if bt > 1 else (M, K)
    shp_b = (bt, K, N) if bt > 1 else (K, N)
    shp_o = (bt, M, N) if bt > 1 else (M, N)
    a = torch.randn(shp_a, device=dev).bfloat16()
    b = torch.randn(shp_b, device=dev).bfloat16()
    o1 = torch.empty(shp_o, device=dev, dtype=torch.bfloat16)
    o2 = torch.empty(shp_o, device=dev, dtype=torch.bfloat16)
    fns = {"bgx": ours(a, b, o1, bt, M, N, K), "cuBLAS": cublas(a, b, o2, bt)}
    if len(sys.argv) > 1 and sys.argv[1] == "cn2":
        fns["bgx cn2"] = ours(a, b, o1, bt, M, N, K, cn=2)
    for fn in fns.values():
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    flop = 2 * bt * M * N * K
    res = {k: {"burst": [], "sus": [], "mhz": []} for k in fns}
    for rnd in range(3):
        order = list(fns) if rnd % 2 == 0 else list(fns)[::-1]
        for k in order:
            res[k]["burst"].append(burst(fns[k]))
            ms, mhz = sustained(fns[k], res[k]["burst"][-1])
            res[k]["sus"].append(ms)
            res[k]["mhz"].append(mhz)
    rel = ((o1.float() - o2.float()).norm() / o2.float().norm()).item()
    for k, r in res.items():
        b_ms, s_ms = statistics.median(r["burst"]), statistics.median(r["sus"])
        mhz = statistics.median(r["mhz"])
        tf_s = flop / s_ms / 1e9
        print(f"{name:24s} {k:8s} burst {b_ms*1e3:9.1f} us {flop/b_ms/1e9:7.1f} TF | sustained {s_ms*1e3:9.1f} us "
              f"{tf_s:7.1f} TF at {mhz:6.0f} MHz = {tf_s / (mhz / 1e3):6.1f} TF/GHz", flush=True)
    print(f"{name:24s} relF(bgx vs cuBLAS) {rel:.2e}", flush=True)

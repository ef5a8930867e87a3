"""Sustained-load comparison: our tcgen05 GEMM vs cuBLAS on the chain GEMM
shape — per-launch time, SM clock and board power sampled by NVML."""
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml  # noqa: E402
import torch  # noqa: E402

from paper_2503_04771_b200 import _lib  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
dev = torch.device("cuda", 0)
M, N, K = 32768, 8192, 8192
a = torch.randn(M, K, device=dev).bfloat16()
b = torch.randn(K, N, device=dev).bfloat16()
out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
lib = _lib.load()


def ours(cg, raster=0):
    d = _lib.BgxContractDesc()
    d.batch, d.M, d.N, d.K = 1, M, N, K
    d.a, d.b, d.out = a.data_ptr(), b.data_ptr(), out.data_ptr()
    d.a_stride[:] = [0, K, 1]
    d.b_stride[:] = [0, N, 1]
    d.o_stride[:] = [0, N, 1]
    d.in_dtype = d.out_dtype = _lib.BF16
    d.mode = _lib.MODE_TC
    d.sched.cta_group, d.sched.tile_n, d.sched.raster = cg, 256, raster
    sp = torch.cuda.current_stream().cuda_stream
    return lambda: lib.bgx_contract(d, sp)


def run(name, fn, seconds=2.5):
    samples = []
    stop = threading.Event()

    def sampler():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
            time.sleep(0.01)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    th = threading.Thread(target=sampler)
    th.start()
    evs = []
    t0 = time.time()
    while time.time() - t0 < seconds:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        evs.append((e0, e1))
        if len(evs) % 50 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = [x.elapsed_time(y) for x, y in evs[len(evs) // 3:]]
    clk = [c for c, p in samples[len(samples) // 3:]]
    pw = [p for c, p in samples[len(samples) // 3:]]
    print(f"{name}: {statistics.median(ms):.3f} ms {2*M*N*K/statistics.median(ms)/1e9:.0f} TFLOP/s "
          f"sm_clk {statistics.median(clk)} MHz power {statistics.median(pw):.0f} W ({len(ms)} launches)",
          flush=True)
    time.sleep(2.0)


for rep in range(2):
    run("cuBLAS", lambda: torch.matmul(a, b, out=out))
    run("ours cg=2", ours(2))
    run("ours cg=1", ours(1))
    run("ours cg=1 raster16", ours(1, 16))

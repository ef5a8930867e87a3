"""Our tcgen05 GEMM (contract(), automatic tile choice) vs cuBLAS
(torch.matmul) on the BASELINE GEMM shapes, interleaved A/B/A/B so that the
board's power/thermal state affects both alike.  Two regimes per shape:
burst (1 s idle, then 20 timed launches) and sustained (launch back to back
for ~2 s, median of the last half); NVML SM clock sampled during sustained.
One JSON line per (shape, impl, regime, repeat)."""
import json
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml  # noqa: E402
import torch  # noqa: E402

from paper_2503_04771_b200.api import contract  # noqa: E402

pynvml.nvmlInit()
H = pynvml.nvmlDeviceGetHandleByIndex(0)
dev = torch.device("cuda", 0)

SHAPES = {"c4_4096": (1, 4096, 4096, 4096), "c3_b64_1024": (64, 1024, 1024, 1024),
          "8192cube": (1, 8192, 8192, 8192), "c5_chain_gemm": (1, 32768, 8192, 8192)}


def timed(fn, n):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(n)]
    for s, e in ev:
        s.record()
        fn()
        e.record()
    torch.cuda.synchronize()
    return [s.elapsed_time(e) for s, e in ev]


def sustained(fn, seconds=2.0):
    clocks, stop = [], threading.Event()

    def sampler():
        while not stop.is_set():
            clocks.append(pynvml.nvmlDeviceGetClockInfo(H, pynvml.NVML_CLOCK_SM))
            time.sleep(0.01)
    th = threading.Thread(target=sampler)
    th.start()
    ts, t0 = [], time.time()
    while time.time() - t0 < seconds:
        ts += timed(fn, 20)
    stop.set()
    th.join()
    half = ts[len(ts) // 2:]
    return statistics.median(half), statistics.median(clocks[len(clocks) // 2:] or [0])


def main():
    for name, (bt, M, N, K) in SHAPES.items():
        shp_a = (bt, M, K) if bt > 1 else (M, K)
        shp_b = (bt, K, N) if bt > 1 else (K, N)
        a = torch.randn(shp_a, device=dev).bfloat16()
        b = torch.randn(shp_b, device=dev).bfloat16()
        out = torch.empty((bt, M, N) if bt > 1 else (M, N), device=dev, dtype=torch.bfloat16)
        spec = "(b,i,k),(b,k,j)->(b,i,j)" if bt > 1 else "(i,k),(k,j)->(i,j)"
        impls = {"ours": lambda: contract(spec, a, b, out=out),
                 "cublas": lambda: torch.matmul(a, b, out=out)}
        flop = 2 * bt * M * N * K
        for rep in range(2):
            for impl in (["ours", "cublas"] if rep == 0 else ["cublas", "ours"]):
                fn = impls[impl]
                for _ in range(3):
                    fn()
                torch.cuda.synchronize()
                time.sleep(1.0)
                burst = statistics.median(timed(fn, 20))
                sus, mhz = sustained(fn)
                print(json.dumps({"shape": name, "impl": impl, "rep": rep,
                                  "burst_ms": round(burst, 4),
                                  "burst_tflops": round(flop / burst / 1e9, 1),
                                  "sustained_ms": round(sus, 4),
                                  "sustained_tflops": round(flop / sus / 1e9, 1),
                                  "sustained_sm_mhz": mhz}), flush=True)
        del a, b, out


if __name__ == "__main__":
    main()

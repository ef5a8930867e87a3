"""A/B two builds of libbgx.so in ONE process (both loaded with ctypes,
RTLD_LOCAL) plus cuBLAS, interleaved, on the BASELINE GEMM shapes: burst
(after 1 s idle, median of 20) and sustained (~2 s back to back, median of
the second half) with the NVML SM clock.  Usage:
    python scripts/ab_lib.py NEW.so OLD.so [shape,shape...]
(AB_SCHED="tile_n=512,cta_group=2" forces a schedule on both builds.)
"""
import ctypes
import json
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
H = pynvml.nvmlDeviceGetHandleByIndex(0)
dev = torch.device("cuda", 0)
SHAPES = {"c4_4096": (1, 4096, 4096, 4096), "c3_b64_1024": (64, 1024, 1024, 1024),
          "8192cube": (1, 8192, 8192, 8192), "c5_chain_gemm": (1, 32768, 8192, 8192)}


def load(path):
    lib = ctypes.CDLL(os.path.abspath(path))
    for name, (res, args) in _lib.SIGNATURES.items():
        fn = getattr(lib, name, None)   # an older build may lack newer entry points
        if fn is not None:
            fn.restype, fn.argtypes = res, args
    return lib


def launcher(lib, a, b, out, bt, M, N, K):
    d = _lib.BgxContractDesc()
    d.batch, d.M, d.N, d.K = bt, M, N, K
    d.a, d.b, d.out = a.data_ptr(), b.data_ptr(), out.data_ptr()
    d.a_stride[:] = [M * K, K, 1]
    d.b_stride[:] = [K * N, N, 1]
    d.o_stride[:] = [M * N, N, 1]
    d.in_dtype = d.out_dtype = _lib.BF16
    d.mode = _lib.MODE_TC
    sched = os.environ.get("AB_SCHED")   # e.g. "tile_n=512,cta_group=2"
    if sched:
        from paper_2503_04771_b200.schedule import Schedule
        for k, v in Schedule.parse(sched).to_dict().items():
            if k == "cluster_n":
                d.sched.reserved[1] = v
            elif k != "splits":
                setattr(d.sched, k, v)
    st = torch.cuda.current_stream().cuda_stream

    def run():
        rc = lib.bgx_contract(d, st)
        assert rc == 0, lib.bgx_last_error()
    return run


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
    return statistics.median(ts[len(ts) // 2:]), statistics.median(clocks[len(clocks) // 2:] or [0])


def main():
    new, old = load(sys.argv[1]), load(sys.argv[2])
    shapes = sys.argv[3].split(",") if len(sys.argv) > 3 else list(SHAPES)
    for name in shapes:
        bt, M, N, K = SHAPES[name]
        a = torch.randn(bt, M, K, device=dev).bfloat16()
        b = torch.randn(bt, K, N, device=dev).bfloat16()
        out = torch.empty(bt, M, N, device=dev, dtype=torch.bfloat16)
        impls = {"new": launcher(new, a, b, out, bt, M, N, K),
                 "old": launcher(old, a, b, out, bt, M, N, K),
                 "cublas": lambda: torch.matmul(a, b, out=out)}
        flop = 2 * bt * M * N * K
        for order in (["new", "old", "cublas"], ["cublas", "old", "new"]):
            for impl in order:
                fn = impls[impl]
                for _ in range(3):
                    fn()
                torch.cuda.synchronize()
                time.sleep(1.0)
                burst = statistics.median(timed(fn, 20))
                sus, mhz = sustained(fn)
                print(json.dumps({"shape": name, "impl": impl, "burst_tflops":
                                  round(flop / burst / 1e9, 1), "sustained_tflops":
                                  round(flop / sus / 1e9, 1), "sustained_sm_mhz": mhz}), flush=True)
        del a, b, out


if __name__ == "__main__":
    main()

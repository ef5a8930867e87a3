"""Per-rank work of the M-sharded chain at N = 1, 2, 4, 8 GPUs, timed on ONE
B200 (each rank's step has no collective, so the N-GPU step time is the max
of N such independent times): projected aggregate TFLOP/s and strong-scaling
efficiency from single-GPU measurements.  Interleaved over N, 2 rounds."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200 import executor, shard  # noqa: E402

dev = torch.device("cuda", 0)
I, K, J, L = 32768, 8192, 8192, 8192
B = torch.randn(K, J, device=dev).bfloat16()
C = torch.randn(J, L, device=dev).bfloat16()
A = torch.randn(I, K, device=dev).bfloat16()
T = torch.empty(I, J, device=dev, dtype=torch.bfloat16)
O = torch.empty(I, L, device=dev, dtype=torch.bfloat16)
flop = 2 * I * J * (K + L)


def step(rows):
    executor.contract_raw(A, (0, K, 1), B, (0, J, 1), T, (0, J, 1), batch=1, M=rows, N=J, K=K,
                          mode="tc")
    executor.contract_raw(T, (0, J, 1), C, (0, L, 1), O, (0, L, 1), batch=1, M=rows, N=L, K=J,
                          mode="tc")


res = {}
for rnd in range(2):
    for n in (1, 2, 4, 8):
        r0, r1 = shard.row_range(I, n, 0)
        rows = r1 - r0
        for _ in range(3):
            step(rows)
        torch.cuda.synchronize()
        time.sleep(1.0)   # same idle before every measurement (power state)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 4 * n
        s.record()
        for _ in range(reps):
            step(rows)
        e.record()
        torch.cuda.synchronize()
        res.setdefault(n, []).append(s.elapsed_time(e) / reps)
base = statistics.mean(res[1])
for n in (1, 2, 4, 8):
    ms = statistics.mean(res[n])
    print(json.dumps({"n_gpus": n, "rows_per_rank": shard.row_range(I, n, 0)[1],
                      "ms_per_rank_step": round(ms, 4), "projected_tflops": round(flop / ms / 1e9, 1),
                      "projected_speedup": round(base / ms, 2),
                      "projected_efficiency": round(base / ms / n, 3)}), flush=True)

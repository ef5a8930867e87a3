"""Interleaved A/B of schedules through contract() (includes split-K /
tail-split workspaces): python scripts/ab_contract.py MxNxK "sched1" "sched2" ...
("" = automatic).  Median of 20 launches per round, 3 rounds."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200 import executor  # noqa: E402
from paper_2503_04771_b200.api import contract  # noqa: E402
from paper_2503_04771_b200.schedule import as_schedule_dict  # noqa: E402

dev = torch.device("cuda", 0)
M, N, K = (int(x) for x in sys.argv[1].split("x"))
a = torch.randn(M, K, device=dev).bfloat16()
b = torch.randn(K, N, device=dev).bfloat16()
out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
scheds = sys.argv[2:] or [""]
res = {s: [] for s in scheds}
kinds = {}
for rnd in range(3):
    for s in (scheds if rnd % 2 == 0 else scheds[::-1]):
        sc = as_schedule_dict(s) if s else None
        for _ in range(3):
            contract("(i,k),(k,j)->(i,j)", a, b, out=out, schedule=sc)
        torch.cuda.synchronize()
        time.sleep(1.0)   # same idle before every measurement (power state)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(20)]
        for e0, e1 in ev:
            e0.record()
            contract("(i,k),(k,j)->(i,j)", a, b, out=out, schedule=sc)
            e1.record()
        torch.cuda.synchronize()
        res[s].append(2 * M * N * K / statistics.median(x.elapsed_time(y) for x, y in ev) / 1e9)
        executor.reset_launch_log()
        contract("(i,k),(k,j)->(i,j)", a, b, out=out, schedule=sc)
        kinds[s] = executor.launch_log()[-1]
for s in scheds:
    print(f"{M}x{N}x{K} [{s or 'auto'}] {kinds[s]}: " + " ".join(f"{v:.0f}" for v in res[s]) + " TFLOP/s",
          flush=True)

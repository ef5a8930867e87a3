"""Per-kernel device times of one contract() call (torch.profiler, CUDA
activities).  python scripts/r02/prof_one.py SPEC a=..,b=.. [mode] [dtype]"""
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_2503_04771_b200 import contract  # noqa: E402

dev = torch.device("cuda", 0)
spec = sys.argv[1]
ext = {k: int(v) for k, v in (kv.split("=") for kv in sys.argv[2].split(","))}
mode = sys.argv[3] if len(sys.argv) > 3 else "auto"
dt = getattr(torch, sys.argv[4]) if len(sys.argv) > 4 else torch.float32
ins, out = spec.split("->")
tups = [t.strip("()").split(",") for t in ins.split("),(")]
otup = [x for x in out.strip("()").split(",") if x]
xs = [torch.randn([ext[a] for a in t], device=dev, dtype=dt) for t in tups]
o = torch.empty([ext[a] for a in otup], device=dev, dtype=dt)
for _ in range(3):
    contract(spec, *xs, out=o, mode=mode)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        contract(spec, *xs, out=o, mode=mode)
    torch.cuda.synchronize()
print(spec, ext, mode, str(dt)[6:])
for ev in prof.key_averages():
    if ev.device_type.name == "CUDA" and ev.count:
        print(f"   {ev.count:3d} x {ev.device_time_total / ev.count:9.1f} us  {ev.key[:90]}")

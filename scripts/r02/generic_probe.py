"""Time one exact generic body (default: the perf-fuzz outlier
(a,d,c),(b)->(d,a,c) f32, a=d=1024, c=b=64) and print the kernels used."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_04771_b200 import contract, executor  # noqa: E402

dev = torch.device("cuda", 0)
spec = sys.argv[1] if len(sys.argv) > 1 else "(a,d,c),(b)->(d,a,c)"
ext = dict(a=1024, d=1024, c=64, b=64)
if len(sys.argv) > 2:
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
executor.reset_launch_log()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    contract(spec, *xs, out=o, mode=mode)
e1.record()
torch.cuda.synchronize()
print(spec, ext, mode, str(dt)[6:], f"{e0.elapsed_time(e1) / 5 * 1e3:.1f} us", executor.launch_log()[:3])

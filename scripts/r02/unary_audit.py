"""One-input bodies (permutations, reductions) over layouts and dtypes: time
vs bytes / 6.5 TB/s (every kernel here is memory-bound except the exact
reference-order chains); flags runs under 25 % of that bound."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_04771_b200 import contract, executor  # noqa: E402

dev = torch.device("cuda", 0)
CASES = [
    ("(a,b)->(b,a)", dict(a=8191, b=8193)),
    ("(a,b)->(b,a)", dict(a=65536, b=1024)),
    ("(a,b)->(b,a)", dict(a=1024, b=65536)),
    ("(a,b,c)->(c,b,a)", dict(a=255, b=513, c=511)),
    ("(a,b,c)->(a,c,b)", dict(a=1024, b=256, c=256)),
    ("(a,b,c)->(b,a,c)", dict(a=256, b=1024, c=256)),
    ("(a,b,c,d)->(d,c,b,a)", dict(a=64, b=64, c=64, d=64)),
    ("(a,b,c,d)->(b,d,a,c)", dict(a=32, b=64, c=128, d=64)),
    ("(a,b)->(a)", dict(a=16384, b=4096)),
    ("(a,b)->(b)", dict(a=16384, b=4096)),
    ("(a,b,c)->(a,c)", dict(a=256, b=512, c=512)),
    ("(a,b,c)->(b)", dict(a=256, b=512, c=512)),
    ("(a,b,c)->(c,a)", dict(a=256, b=512, c=512)),
]
for dt in (torch.float32, torch.bfloat16):
    for spec, ext in CASES:
        ins, out = spec.split("->")
        tup = ins.strip("()").split(",")
        otup = [x for x in out.strip("()").split(",") if x]
        x = torch.randn([ext[a] for a in tup], device=dev).to(dt)
        o = torch.empty([ext[a] for a in otup], device=dev, dtype=dt)
        f = lambda: contract(spec, x, out=o)  # noqa: E731
        for _ in range(2):
            f()
        torch.cuda.synchronize()
        executor.reset_launch_log()
        f()
        kinds = executor.launch_log()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); f(); e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        byts = (x.numel() + o.numel()) * x.element_size()
        bound = byts / 6.5e12 * 1e3
        frac = bound / ms
        flag = "SLOW" if frac < 0.25 else "    "
        print(f"{flag} {str(dt)[6:]:9s} {spec:22s} {str(ext):40s} {ms*1e3:9.1f} us  bound {bound*1e3:7.1f} us "
              f"({100*frac:5.1f} %)  {kinds[:2]}", flush=True)

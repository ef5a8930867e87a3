"""Two-operand contraction shapes a user might hit (tall/skinny, tiny N,
outer products, transposed outputs, batched) in bf16 (tensor cores) and f32
(exact): time against a simple roofline (max of bytes / 6.5 TB/s and
flop / peak, peak = 1600 TFLOP/s bf16 or 36 TFLOP/s f32 exact) and the kernel
picked; flags runs under 20 % of that bound."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_04771_b200 import contract, executor, plan  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] == "off":
    plan.OUTER_TO_LOOP_NEST = plan.SKINNY_TO_LOOP_NEST = False

dev = torch.device("cuda", 0)
CASES = [
    ("(i,k),(k,j)->(i,j)", dict(i=1 << 20, k=64, j=8)),
    ("(i,k),(k,j)->(i,j)", dict(i=8, k=64, j=1 << 20)),
    ("(i,k),(k,j)->(i,j)", dict(i=1 << 18, k=256, j=64)),
    ("(i,k),(k,j)->(i,j)", dict(i=64, k=1 << 20, j=64)),
    ("(i,k),(k,j)->(i,j)", dict(i=16, k=4096, j=16384)),
    ("(i),(j)->(i,j)", dict(i=8192, j=8192)),
    ("(i,k),(k,j)->(j,i)", dict(i=4096, k=4096, j=4096)),
    ("(i,k),(j,k)->(i,j)", dict(i=4096, k=4096, j=4096)),
    ("(k,i),(k,j)->(i,j)", dict(i=4096, k=4096, j=4096)),
    ("(b,i,k),(b,k,j)->(b,i,j)", dict(b=512, i=64, k=64, j=64)),
    ("(b,i,k),(k,j)->(b,i,j)", dict(b=64, i=512, k=512, j=512)),
    ("(i,b,k),(b,k,j)->(b,i,j)", dict(b=32, i=512, k=512, j=512)),
]
for dt, peak in ((torch.bfloat16, 1600e12), (torch.float32, 36e12)):
    for spec, ext in CASES:
        ins, out = spec.split("->")
        tups = [t.strip("()").split(",") for t in ins.split("),(")]
        otup = [x for x in out.strip("()").split(",") if x]
        xs = [torch.randn([ext[a] for a in t], device=dev).to(dt) for t in tups]
        o = torch.empty([ext[a] for a in otup], device=dev, dtype=dt)
        f = lambda: contract(spec, *xs, out=o)  # noqa: E731
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
        pts = 1
        for v in ext.values():
            pts *= v
        byts = (sum(x.numel() for x in xs) + o.numel()) * o.element_size()
        bound = max(byts / 6.5e12, 2 * pts / peak) * 1e3
        frac = bound / ms
        flag = "SLOW" if frac < 0.2 else "    "
        print(f"{flag} {str(dt)[6:]:9s} {spec:26s} {str(ext):42s} {ms*1e3:9.1f} us  bound {bound*1e3:8.1f} us "
              f"({100*frac:5.1f} %)  {kinds[:3]}", flush=True)

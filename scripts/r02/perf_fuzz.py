"""Random einsum bodies at sizes of 16-256 MB of operand traffic, auto mode,
f32 and bf16: flags plans far below both the HBM and the tensor roofline
(effective GB/s < 500 and TFLOP/s < 50), printing the kernels used."""
import random
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2503_04771_b200 import contract, executor  # noqa: E402
from paper_2503_04771_b200 import einsum as E  # noqa: E402

dev = torch.device("cuda", 0)
r = random.Random(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
letters = ["a", "b", "c", "d"]
n = 0
flagged = 0
while n < int(sys.argv[2]) if len(sys.argv) > 2 else 60:
    ins = [tuple(r.sample(letters, r.randint(1, 3))) for _ in range(r.randint(1, 3))]
    used = sorted({x for t in ins for x in t})
    out = tuple(r.sample(used, r.randint(0, min(3, len(used)))))
    text = ",".join("(" + ",".join(t) + ")" for t in ins) + "->(" + ",".join(out) + ")"
    try:
        spec = E.parse_einsum(text)
    except E.EinsumError:
        continue
    # extents so that the largest operand/output is 4-64 M elements
    ext = {a: r.choice([8, 64, 256, 1024, 4096]) for a in spec.axes}
    sizes = [int(np.prod([ext[a] for a in t])) for t in (*spec.inputs, spec.output)]
    pts = int(np.prod([ext[a] for a in spec.axes]))
    if max(sizes) < (1 << 22) or max(sizes) > (1 << 26) or pts > (1 << 34):
        continue
    for dt in (torch.float32, torch.bfloat16):
        if dt == torch.float32 and len(spec.inputs) >= 3 and pts > (1 << 28):
            continue        # the exact 3-operand loop nest: reference order, slow by design
        xs = [torch.randn([ext[a] for a in t], device=dev).to(dt) for t in spec.inputs]
        o = torch.empty([ext[a] for a in spec.output], device=dev, dtype=dt)
        try:
            contract(spec, *xs, out=o)
        except Exception as e:  # noqa: BLE001
            print(f"ERROR {text} {ext} {dt}: {type(e).__name__}: {e}"[:200], flush=True)
            continue
        executor.reset_launch_log()
        contract(spec, *xs, out=o)
        kern = sorted(set(executor.launch_log()))
        ts = []
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            contract(spec, *xs, out=o)
            b.record()
            ts.append((a, b))
        torch.cuda.synchronize()
        ms = statistics.median(x.elapsed_time(y) for x, y in ts)
        nb = sum(x.numel() * x.element_size() for x in xs) + o.numel() * o.element_size()
        gbs, tfs = nb / ms / 1e6, 2 * pts / ms / 1e9
        red = pts // max(1, o.numel())
        exact_chain = dt == torch.float32 and red >= 4096      # reference order, by design
        bad = gbs < 500 and tfs < 50 and not exact_chain
        flagged += bad
        print(f"{'SLOW ' if bad else '     '}{text:34s} {str(ext):48s} {str(dt)[6:]:9s} {ms*1e3:10.1f} us "
              f"{gbs:7.0f} GB/s {tfs:7.2f} TF/s red={red} {kern}", flush=True)
    n += 1
print("flagged", flagged)

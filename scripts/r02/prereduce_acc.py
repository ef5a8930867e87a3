"""Accuracy of the 16-bit pre-reduction at a given blow-up threshold
(executor.PREREDUCE_16BIT_BLOWUP): random bodies with private reduction
axes, bf16, auto mode, relF vs float64 einsum of the same bf16 values."""
import random
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2503_04771_b200 import contract, executor  # noqa: E402
from paper_2503_04771_b200 import einsum as E  # noqa: E402

executor.PREREDUCE_16BIT_BLOWUP = int(sys.argv[1]) if len(sys.argv) > 1 else 64
dev = torch.device("cuda", 0)
r = random.Random(99)
nr = np.random.default_rng(99)
letters = ["a", "b", "c", "d"]
worst, n, pre = 0.0, 0, 0
while n < 150:
    ins = [tuple(r.sample(letters, r.randint(1, 3))) for _ in range(r.randint(2, 3))]
    used = sorted({x for t in ins for x in t})
    out = tuple(r.sample(used, r.randint(0, min(2, len(used)))))
    text = ",".join("(" + ",".join(t) + ")" for t in ins) + "->(" + ",".join(out) + ")"
    try:
        spec = E.parse_einsum(text)
    except E.EinsumError:
        continue
    if not executor._private_axes(spec):
        continue
    ext = {a: r.choice([3, 16, 64, 256, 1024]) for a in spec.axes}
    pts = int(np.prod([ext[a] for a in spec.axes]))
    lo_pts = float(sys.argv[2]) if len(sys.argv) > 2 else 1e4
    if pts > 3e8 or pts < lo_pts:
        continue
    xs = [torch.from_numpy(nr.standard_normal(tuple(ext[x] for x in t))).to(dev).bfloat16()
          for t in spec.inputs]
    executor.reset_launch_log()
    got = contract(spec, *xs).double()
    tt = ",".join("".join(t) for t in spec.inputs) + "->" + "".join(spec.output)
    want = torch.einsum(tt, *[x.double() for x in xs])
    err = ((got - want).norm() / (want.norm() + 1e-30)).item()
    size = sum(x.numel() for x in xs)
    used_pre = pts >= executor.PREREDUCE_16BIT_BLOWUP * size
    pre += used_pre
    worst = max(worst, err)
    if err > 1e-2:
        print(f"{text:28s} {ext} relF {err:.2e} prereduced={used_pre} {executor.launch_log()} |want| {want.norm().item():.3g}")
    n += 1
print(f"threshold {executor.PREREDUCE_16BIT_BLOWUP}: {n} bodies, {pre} pre-reduced, worst relF {worst:.2e}")

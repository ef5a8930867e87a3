"""Accuracy envelope of the f32 tolerance mode (mode='ffma': FFMA GEMMs, tree
reductions, f32 pre-reductions and chains): random 1-3 input bodies, relF vs
float64 einsum of the same f32 values; the API promises <= 1e-5."""
import random
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2503_04771_b200 import contract, executor  # noqa: E402
from paper_2503_04771_b200 import einsum as E  # noqa: E402

dev = torch.device("cuda", 0)
r = random.Random(7)
nr = np.random.default_rng(7)
letters = ["a", "b", "c", "d"]
worst, n = 0.0, 0
lo_pts = float(sys.argv[1]) if len(sys.argv) > 1 else 1e4
while n < 150:
    ins = [tuple(r.sample(letters, r.randint(1, 3))) for _ in range(r.randint(1, 3))]
    used = sorted({x for t in ins for x in t})
    out = tuple(r.sample(used, r.randint(0, min(2, len(used)))))
    text = ",".join("(" + ",".join(t) + ")" for t in ins) + "->(" + ",".join(out) + ")"
    try:
        spec = E.parse_einsum(text)
    except E.EinsumError:
        continue
    if len(spec.inputs) == 1 and set(spec.inputs[0]) == set(spec.output):
        continue
    ext = {a: r.choice([3, 16, 64, 256, 1024]) for a in spec.axes}
    pts = int(np.prod([ext[a] for a in spec.axes]))
    if pts > 3e8 or pts < lo_pts:
        continue
    xs = [torch.from_numpy(nr.standard_normal(tuple(ext[x] for x in t))).to(dev).float()
          for t in spec.inputs]
    executor.reset_launch_log()
    got = contract(spec, *xs, mode="ffma").double()
    tt = ",".join("".join(t) for t in spec.inputs) + "->" + "".join(spec.output)
    want = torch.einsum(tt, *[x.double() for x in xs])
    err = ((got - want).norm() / (want.norm() + 1e-30)).item()
    worst = max(worst, err)
    if err > 1e-5:
        print(f"{text:28s} {ext} relF {err:.2e} {executor.launch_log()} |want| {want.norm().item():.3g}")
    n += 1
print(f"ffma: {n} bodies, worst relF {worst:.2e}")

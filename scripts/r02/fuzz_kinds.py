import random, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2503_04771_b200 import contract, executor
from paper_2503_04771_b200 import einsum as E
dev = torch.device("cuda", 0)
r = random.Random(20261019); nr = np.random.default_rng(20261019)
letters = ["a", "b", "c", "d"]; seen = 0; kinds = {}
while seen < 30:
    ins = [tuple(r.sample(letters, r.randint(1, 3))) for _ in range(r.randint(1, 3))]
    used = sorted({x for t in ins for x in t})
    out = tuple(r.sample(used, r.randint(0, min(3, len(used)))))
    text = ",".join("(" + ",".join(t) + ")" for t in ins) + "->(" + ",".join(out) + ")"
    try: spec = E.parse_einsum(text)
    except E.EinsumError: continue
    if len(spec.inputs) == 1 and set(spec.inputs[0]) == set(spec.output): continue
    ext = {a: r.choice([3, 16, 64, 130, 512, 1024]) for a in spec.axes}
    n_out = int(np.prod([ext[a] for a in spec.output])) if spec.output else 1
    pts = int(np.prod([ext[a] for a in spec.axes]))
    if pts > 12_000_000 or pts < 20_000: continue
    arrs = [nr.standard_normal(tuple(ext[x] for x in t)).astype(np.float32) for t in spec.inputs]
    c0 = nr.standard_normal(tuple(ext[x] for x in spec.output)).astype(np.float32)
    executor.reset_launch_log()
    contract(spec, *[torch.from_numpy(a).to(dev) for a in arrs], c0=torch.from_numpy(c0).to(dev), mode="exact")
    print(f"{text:28s} n_out={n_out:9d} pts={pts:9d} {executor.launch_log()}")
    seen += 1

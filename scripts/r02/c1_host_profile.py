"""Where the host time of a replayed run_function call (BASELINE C1) goes."""
import cProfile
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2503_04771_b200 import einsum as E  # noqa: E402
from paper_2503_04771_b200 import interp as I  # noqa: E402

dev = torch.device("cuda", 0)
rng = np.random.default_rng(1)
ts = [torch.from_numpy(rng.standard_normal((256, 256), dtype=np.float32)).to(dev) for _ in range(2)]
ts.append(torch.zeros(256, 256, device=dev))
mod = E.build_einsum_function(None, E.parse_einsum("(i,j),(j,k)->(i,k)"))
vals = [I.TensorValue(E.F32, (256, 256), t) for t in ts]
for _ in range(50):
    I.run_function(mod, "einsum", vals, step_limit=None)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(2000):
    I.run_function(mod, "einsum", vals, step_limit=None)
torch.cuda.synchronize()
print("per call us", (time.perf_counter() - t0) / 2000 * 1e6)
pr = cProfile.Profile()
pr.enable()
for _ in range(2000):
    I.run_function(mod, "einsum", vals, step_limit=None)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)

import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_04771_b200 import einsum as E  # noqa: E402
from paper_2503_04771_b200 import interp as I  # noqa: E402

dev = torch.device("cuda", 0)
rng = np.random.default_rng(1)
xs = [rng.standard_normal((256, 256), dtype=np.float32) for _ in range(2)] + [np.zeros((256, 256), np.float32)]
mod = E.build_einsum_function(None, E.parse_einsum("(i,j),(j,k)->(i,k)"))
vals = [I.TensorValue(E.F32, x.shape, torch.from_numpy(x).to(dev)) for x in xs]
for _ in range(20):
    I.run_function(mod, "einsum", vals, step_limit=None)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(2000):
    I.run_function(mod, "einsum", vals, step_limit=None)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)

"""BASELINE config 1 (256^3 f32 via the reference-shaped API): where the
~70 us per call go — numpy in/out vs device tensors vs prepare()."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_04771_b200 import einsum as E  # noqa: E402
from paper_2503_04771_b200 import interp as I  # noqa: E402
from paper_2503_04771_b200 import prepare  # noqa: E402

dev = torch.device("cuda", 0)
rng = np.random.default_rng(1)
a, b = (rng.standard_normal((256, 256), dtype=np.float32) for _ in range(2))
c = np.zeros((256, 256), np.float32)
mod = E.build_einsum_function(None, E.parse_einsum("(i,j),(j,k)->(i,k)"))
host_vals = [I.TensorValue(E.F32, x.shape, x) for x in (a, b, c)]
dev_vals = [I.TensorValue(E.F32, x.shape, torch.from_numpy(x).to(dev)) for x in (a, b, c)]


def t(fn, n=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    s = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - s) / n * 1e6


print("run_function numpy in/out : %.1f us" % t(lambda: I.run_function(mod, "einsum", host_vals, step_limit=None)))
print("run_function device values: %.1f us" % t(lambda: I.run_function(mod, "einsum", dev_vals, step_limit=None)))
A, B = (torch.from_numpy(x).to(dev) for x in (a, b))
p = prepare("(i,j),(j,k)->(i,k)", A, B)
print("prepare()                 : %.1f us" % t(lambda: p()))
g = prepare("(i,j),(j,k)->(i,k)", A, B, graph=True)
print("prepare(graph=True)       : %.1f us" % t(lambda: g()))

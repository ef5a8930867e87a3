"""BASELINE C1 through the reference-shaped DSL (run_function), device-resident
inputs: host+device time per call (the bench aux number's path)."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_04771_b200 import einsum as E  # noqa: E402
from paper_2503_04771_b200 import interp as I  # noqa: E402

dev = torch.device("cuda", 0)
rng = np.random.default_rng(1)
xs = [torch.from_numpy(rng.standard_normal((256, 256), dtype=np.float32)).to(dev) for _ in range(2)]
xs.append(torch.zeros(256, 256, device=dev))
mod = E.build_einsum_function(None, E.parse_einsum("(i,j),(j,k)->(i,k)"))
vals = [I.TensorValue(E.F32, (256, 256), t) for t in xs]
fn = lambda: I.run_function(mod, "einsum", vals, step_limit=None)  # noqa: E731
for _ in range(20):
    fn()
torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    for _ in range(500):
        fn()
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0) / 500 * 1e6)
print(f"C1 run_function: {statistics.median(ts):.1f} us per call "
      f"({2 * 256 ** 3 / statistics.median(ts) / 1e6:.2f} TFLOP/s)")

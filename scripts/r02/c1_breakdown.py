"""BASELINE config 1 (256^3 f32 exact through the reference-shaped API):
where the per-call time goes."""
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2503_04771_b200 import _lib, contract  # noqa: E402
from paper_2503_04771_b200 import einsum as E  # noqa: E402
from paper_2503_04771_b200 import interp as I  # noqa: E402

dev = torch.device("cuda", 0)
rng = np.random.default_rng(1)
a = torch.from_numpy(rng.standard_normal((256, 256), dtype=np.float32)).to(dev)
b = torch.from_numpy(rng.standard_normal((256, 256), dtype=np.float32)).to(dev)
c = torch.zeros(256, 256, device=dev)
mod = E.build_einsum_function(None, E.parse_einsum("(i,j),(j,k)->(i,k)"))
vals = [I.TensorValue(E.F32, (256, 256), t) for t in (a, b, c)]
out = torch.empty(256, 256, device=dev)
lib = _lib.load()
d = _lib.BgxContractDesc()
d.batch, d.M, d.N, d.K = 1, 256, 256, 256
d.a, d.b, d.out = a.data_ptr(), b.data_ptr(), out.data_ptr()
d.a_stride[:] = [0, 256, 1]
d.b_stride[:] = [0, 256, 1]
d.o_stride[:] = [0, 256, 1]
d.in_dtype = d.out_dtype = _lib.F32
d.mode = _lib.MODE_EXACT
st = torch.cuda.current_stream().cuda_stream
fns = {"raw bgx_contract": lambda: lib.bgx_contract(d, st),
       "contract(mode=exact)": lambda: contract("(i,j),(j,k)->(i,k)", a, b, out=out, mode="exact"),
       "run_function": lambda: I.run_function(mod, "einsum", vals, step_limit=None)}
for name, fn in fns.items():
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    # device time per call, one call at a time (event pair around each)
    evs = []
    for _ in range(200):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    dev_ms = statistics.median(x.elapsed_time(y) for x, y in evs)
    # host wall per call, back to back (pipelined)
    t0 = time.perf_counter()
    for _ in range(2000):
        fn()
    torch.cuda.synchronize()
    wall_us = (time.perf_counter() - t0) / 2000 * 1e6
    # host time to issue one call (no sync)
    t0 = time.perf_counter()
    for _ in range(200):
        fn()
    issue_us = (time.perf_counter() - t0) / 200 * 1e6
    torch.cuda.synchronize()
    print(f"{name:24s} event-pair {dev_ms*1e3:7.1f} us   back-to-back {wall_us:7.1f} us/call   "
          f"host issue {issue_us:7.1f} us", flush=True)

"""How far the persistent CTAs drift apart: start time of every CTA's n-th
unit (static round-robin schedule), spread per wave (schedule debug 4096)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts/r02")
from paper_2503_04771_b200 import _lib  # noqa: E402
from probe_drain import SHAPES  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "chain"
bt, M, N, K = SHAPES[shape]
lib = _lib.load()
dev = torch.device("cuda", 0)
a = torch.randn(bt, M, K, device=dev).bfloat16()
b = torch.randn(bt, K, N, device=dev).bfloat16()
out = torch.empty(bt, M, N, device=dev, dtype=torch.bfloat16)
d = _lib.BgxContractDesc()
d.batch, d.M, d.N, d.K = bt, M, N, K
d.a, d.b, d.out = a.data_ptr(), b.data_ptr(), out.data_ptr()
d.a_stride[:] = [M * K, K, 1]
d.b_stride[:] = [K * N, N, 1]
d.o_stride[:] = [M * N, N, 1]
d.in_dtype = d.out_dtype = _lib.BF16
d.mode = _lib.MODE_TC
d.sched.reserved[0] = 4096
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    _lib.check(lib.bgx_contract(d, st), "c")
torch.cuda.synchronize()
buf = np.zeros(160 * 64, dtype=np.uint64)
f = lib.bgxdbg_trace_read
f.argtypes = [ctypes.c_void_p, ctypes.c_int64]
assert f(buf.ctypes.data, buf.nbytes) == 0
tr = buf.reshape(160, 64).astype(np.int64)
live = tr[:, 0] > 0
tr = tr[live]
t0 = tr[tr > 0].min()
print(shape, "CTAs traced", tr.shape[0])
for w in range(0, 64):
    col = tr[:, w]
    col = col[col > 0]
    if len(col) < 2:
        break
    print(f"unit {w:2d}: start min {(col.min()-t0)/1e3:9.1f} us  max {(col.max()-t0)/1e3:9.1f}  "
          f"spread {(col.max()-col.min())/1e3:7.1f} us  n={len(col)}")

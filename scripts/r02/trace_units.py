"""Per-unit timeline of the first CTAs of one GEMM launch (schedule debug
bit 4096): producer / MMA / epilogue receive the unit, epilogue sees the
accumulator full.  python scripts/r02/trace_units.py SHAPE key=val,..."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts/r02")
from paper_2503_04771_b200 import _lib  # noqa: E402
from probe_drain import SHAPES  # noqa: E402

shape, text = sys.argv[1], sys.argv[2]
kw = dict((k, int(v)) for k, v in (p.split("=") for p in text.split(",") if p))
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
for k, v in kw.items():
    if k == "debug":
        d.sched.reserved[0] = v | 4096
    elif k == "cluster_n":
        d.sched.reserved[1] = v
    else:
        setattr(d.sched, k, v)
if "debug" not in kw:
    d.sched.reserved[0] = 4096
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    _lib.check(lib.bgx_contract(d, st), "c")
torch.cuda.synchronize()
buf = np.zeros(8 * 64 * 4, dtype=np.uint64)
f = lib.bgxdbg_trace_read
f.argtypes = [ctypes.c_void_p, ctypes.c_int64]
assert f(buf.ctypes.data, buf.nbytes) == 0
tr = buf.reshape(8, 64, 4).astype(np.int64)
t0 = tr[tr > 0].min()
print(shape, kw)
for cta in range(8):
    rows = [r for r in tr[cta] if r[0] > 0]
    print(f"CTA {cta}: {len(rows)} units")
    for i, r in enumerate(rows[:20]):
        print("   unit%2d prod %8.2f mma %8.2f epi %8.2f accfull %8.2f us" %
              (i, *((r - t0) / 1e3)))

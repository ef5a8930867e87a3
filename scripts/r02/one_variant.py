"""Run ONE schedule variant of a probe shape a few times (for ncu capture):
python scripts/r02/one_variant.py SHAPE key=val,key=val"""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts/r02")
from paper_2503_04771_b200 import _lib  # noqa: E402
from probe_drain import SHAPES  # noqa: E402

shape, text = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
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
        d.sched.reserved[0] = v
    elif k == "cluster_n":
        d.sched.reserved[1] = v
    else:
        setattr(d.sched, k, v)
st = torch.cuda.current_stream().cuda_stream
for _ in range(4):
    _lib.check(lib.bgx_contract(d, st), "c")
torch.cuda.synchronize()
print("ok", shape, kw)

import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2503_04771_b200 import _lib  # noqa: E402
dev = torch.device("cuda", 0)
lib = _lib.load()
M = N = K = int(sys.argv[1]) if len(sys.argv) > 1 else 256
a = torch.randn(M, K, device=dev); b = torch.randn(K, N, device=dev); out = torch.empty(M, N, device=dev)
d = _lib.BgxContractDesc()
d.batch, d.M, d.N, d.K = 1, M, N, K
d.a, d.b, d.out = a.data_ptr(), b.data_ptr(), out.data_ptr()
d.a_stride[:] = [0, K, 1]; d.b_stride[:] = [0, N, 1]; d.o_stride[:] = [0, N, 1]
d.in_dtype = d.out_dtype = _lib.F32
d.mode = _lib.MODE_EXACT
st = torch.cuda.current_stream().cuda_stream
for _ in range(30):
    lib.bgx_contract(d, st)
torch.cuda.synchronize()

"""Where does tf32x3's error come from?  Split with bgx_tf32_split, then
(1) multiply the split operands in f64 (the split's own error), (2) run the
tcgen05 tf32 GEMM on them (the tensor-core accumulation's error)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_04771_b200 import _lib, contract, executor  # noqa: E402

dev = torch.device("cuda", 0)
lib = _lib.load()
for n in (1024, 4096):
    a = torch.randn(n, n, device=dev)
    b = torch.randn(n, n, device=dev)
    ref = a.double() @ b.double()
    seg = n
    a2 = torch.empty((1, n, 3 * seg), device=dev)
    b2 = torch.empty((1, 3 * seg, n), device=dev)
    st = torch.cuda.current_stream().cuda_stream
    _lib.check(lib.bgx_tf32_split(a.data_ptr(), 1, n, n, (_lib._i64 * 3)(0, n, 1), a2.data_ptr(),
                                  n * 3 * seg, 3 * seg, 0, seg, st), "split a")
    _lib.check(lib.bgx_tf32_split(b.data_ptr(), 1, n, n, (_lib._i64 * 3)(0, n, 1), b2.data_ptr(),
                                  3 * seg * n, n, 1, seg, st), "split b")
    torch.cuda.synchronize()
    hi = a2[0, :, :seg]
    lo = a2[0, :, 2 * seg:]
    print(n, "a hi low bits zero:", bool(((hi.view(torch.int32) & 0x1FFF) == 0).all()),
          "lo low bits zero:", bool(((lo.view(torch.int32) & 0x1FFF) == 0).all()),
          "hi+lo vs a max rel:", (((hi.double() + lo.double()) - a.double()).abs() / a.double().abs().clamp_min(1e-30)).max().item())
    f64 = a2[0].double() @ b2[0].double()
    print(n, "split operands in f64: relF", ((f64 - ref).norm() / ref.norm()).item())
    o = torch.empty(n, n, device=dev)
    contract("(i,k),(k,j)->(i,j)", a2[0], b2[0], out=o, mode="tf32")
    print(n, "split operands on tcgen05 tf32: relF", ((o.double() - ref).norm() / ref.norm()).item())
    # accumulation alone: exactly-representable tf32 inputs, no split
    at = a2[0, :, :seg].contiguous()
    bt = b2[0, :seg, :].contiguous()
    ref2 = at.double() @ bt.double()
    contract("(i,k),(k,j)->(i,j)", at, bt, out=o, mode="tf32")
    print(n, "tf32-exact inputs, tcgen05 tf32 accumulate: relF", ((o.double() - ref2).norm() / ref2.norm()).item())
    ab = at.bfloat16()
    contract("(i,k),(k,j)->(i,j)", a.bfloat16(), b.bfloat16(), out=o)
    ref3 = a.bfloat16().double() @ b.bfloat16().double()
    print(n, "bf16 inputs, tcgen05 f32 accumulate: relF", ((o.double() - ref3).norm() / ref3.norm()).item())

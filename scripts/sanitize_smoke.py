"""Small invocation of every kernel class (for compute-sanitizer memcheck).

compute-sanitizer is refused on the GPU pool (profiles/r02_sanitizer.txt);
tests/test_gpu_guard_zones.py is the in-repo substitute: the same kernel
classes with NaN-filled guard zones around every operand and a sentinel
pattern around every output."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_04771_b200 import contract  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)


def r(*s, dt=torch.float32):
    return torch.randn(*s, generator=g, device=dev).to(dt)


contract("(i,j)->(j,i)", r(200, 136))                                  # vec transpose
contract("(i,j,k)->(k,i,j)", r(5, 33, 7))                              # generic transpose
contract("(i,j)->(i)", r(50, 77))                                      # generic reduction
contract("(i,j),(j,k),(k,l)->(i,l)", r(9, 10), r(10, 11), r(11, 12))   # generic 3-operand
contract("(i,k),(k,j)->(i,j)", r(300, 200), r(200, 260))               # SIMT exact (64x64)
contract("(i,k),(k,j)->(i,j)", r(1300, 200), r(200, 1260), mode="ffma")  # SIMT big
for cg, bn in ((1, 64), (1, 256), (2, 256), (2, 512)):
    contract("(i,k),(k,j)->(i,j)", r(300, 640, dt=torch.bfloat16), r(640, 1100 - 12, dt=torch.bfloat16),
             schedule={"cta_group": cg, "tile_n": bn})
contract("(b,i,j),(b,j,k)->(b,i,k)", r(3, 130, 72, dt=torch.float16), r(3, 72, 200, dt=torch.float16),
         out_dtype=torch.float32)
contract("(i,k),(k,j)->(i,j)", r(128, 16384, dt=torch.bfloat16), r(16384, 128, dt=torch.bfloat16))  # split-K
contract("(i,k),(j,k)->(i,j)", r(200, 96), r(136, 96), mode="tf32")
try:
    sys.path.append(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref"))
    from bridgegen import interp, ir  # noqa: E402
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden"))
    import make_golden as M  # noqa: E402
    from paper_2503_04771_b200 import fir_gpu  # noqa: E402
    mod = M.pipeline(M.VADD_FIR, "vadd")
    bufs = [interp.MemRefValue(ir.F32, (8,), np.arange(8, dtype=np.float32)) for _ in range(3)]
    fir_gpu.run_kernel(mod, "vadd", interp.LaunchConfig((2, 1, 1), (4, 1, 1)), bufs)
except ImportError as e:
    print("bridgegen not importable, skipping FIR kernel:", e)
# round 2 kernels
contract("(i,j),(i,j)->(i,j)", r(300, 136), r(300, 136))                       # dense_ew (vector)
contract("(i,j),(i,j)->(i,j)", r(301, 137), r(301, 137))                       # dense_ew tail
contract("(i,j)->(i)", r(700, 4096))                                           # rowreduce VEC thin
contract("(i,j)->(i)", r(20000, 96))                                           # rowreduce VEC 4-warp
contract("(i,j)->()", r(3000, 700), mode="ffma")                               # tree contig + finish
contract("(i,j)->(i)", r(3000, 700), mode="ffma")                              # tree contig warp
contract("(i,j)->(j)", r(3000, 700), mode="ffma")                              # tree column
contract("(i,j)->(j)", r(3000, 702, dt=torch.bfloat16))                        # tree column2 (16-bit)
contract("(k),(k,j)->(j)", r(3000, dt=torch.bfloat16), r(3000, 702, dt=torch.bfloat16))
contract("(i,j,k)->(j)", r(40, 37, 300), mode="ffma")                          # tree general
contract("(c,a,b)->(a,c,b)", r(70, 90, 64))                                    # short-row copy
contract("(i)->(i)", r(1 << 20))                                               # chunked row copy
contract("(i,k),(k,j)->(i,j)", r(1000, 320, dt=torch.bfloat16), r(320, 272, dt=torch.bfloat16),
         devices=[0, 0])                                                       # bgx_contract_sharded
torch.cuda.synchronize()
print("sanitize smoke done")

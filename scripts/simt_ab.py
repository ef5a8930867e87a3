"""A/B the f32 SIMT GEMM kernels in one process: the cp.async pipeline 
(2 stages) vs the register-staged kernel
(BGX_NO_SIMT_CP=1); both variables are read at every launch.  Interleaved, median of 7."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_04771_b200.api import contract  # noqa: E402

dev = torch.device("cuda", 0)
MM = "(i,k),(k,j)->(i,j)"
for (m, n, k) in ((2048, 2048, 2048), (4096, 4096, 4096), (1000, 1000, 1000), (8192, 8192, 2048)):
    a = torch.randn(m, k, device=dev)
    b = torch.randn(k, n, device=dev)
    ref = {}
    for rep in range(2):
        for impl in (("cp2", "reg") if rep == 0 else ("reg", "cp2")):
            os.environ.pop("BGX_NO_SIMT_CP", None)
            os.environ["BGX_SIMT_CP_STAGES"] = impl[-1]
            if impl == "reg":
                os.environ["BGX_NO_SIMT_CP"] = "1"
            for mode in ("ffma", "exact"):
                for _ in range(2):
                    o = contract(MM, a, b, mode=mode)
                torch.cuda.synchronize()
                ref.setdefault((mode, impl), o.clone())
                time.sleep(0.3)
                ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                      for _ in range(7)]
                for s, e in ev:
                    s.record(); contract(MM, a, b, mode=mode); e.record()
                torch.cuda.synchronize()
                ms = statistics.median(s.elapsed_time(e) for s, e in ev)
                print(f"{m}x{n}x{k} {mode} {impl} rep{rep}: {ms:.3f} ms "
                      f"{2*m*n*k/ms/1e9:.1f} TFLOP/s", flush=True)
    for mode in ("ffma", "exact"):
        same = all(torch.equal(ref[(mode, c)], ref[(mode, "reg")]) for c in ("cp2",))
        print(f"{m}x{n}x{k} {mode} cp==reg bitwise: {same}", flush=True)

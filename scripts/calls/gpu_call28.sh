#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x --timeout 300 -k "tf32 or fp32 or f64 or c1" > gpurun_out/t_26.log 2>&1; echo "tf32 tests rc=$?"; tail -3 gpurun_out/t_26.log
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/t_26b.log 2>&1; echo "all rc=$?"; tail -2 gpurun_out/t_26b.log
python - <<'PY'
import torch, statistics, sys
sys.path.insert(0, '.')
from paper_2503_04771_b200 import contract
dev = torch.device('cuda', 0)
for (M, N, K) in [(4096, 4096, 4096), (8192, 8192, 8192)]:
    a = torch.randn(M, K, device=dev); b = torch.randn(K, N, device=dev)
    for mode in ("tf32", "ffma"):
        f = lambda: contract('(i,k),(k,j)->(i,j)', a, b, mode=mode)
        for _ in range(2): f()
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        print(f"f32 {M}^3 mode={mode}: {ms:.3f} ms {2*M*N*K/ms/1e9:.0f} TFLOP/s")
PY

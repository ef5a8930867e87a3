#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_edges.py -q -x --timeout 180 > gpurun_out/t_24.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_24.log
python - <<'PY'
import torch, statistics, sys
sys.path.insert(0, '.')
from paper_2503_04771_b200 import contract
dev = torch.device('cuda', 0)
for (M, N, K) in [(256, 256, 1 << 20), (1024, 1024, 1 << 18), (512, 2048, 65536)]:
    a = torch.randn(M, K, device=dev).bfloat16(); b = torch.randn(K, N, device=dev).bfloat16()
    for sched in ({"no_splitk": 1}, None):
        f = lambda: contract('(i,k),(k,j)->(i,j)', a, b, schedule=sched)
        for _ in range(3): f()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        print(f"{M}x{N}x{K} {'no-split' if sched else 'auto   '}: {ms:.3f} ms {2*M*N*K/ms/1e9:.0f} TFLOP/s")
    ms = statistics.median([0])
PY

#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x --timeout 120 > gpurun_out/t_gemm3.log 2>&1; echo "gemm rc=$?"; tail -3 gpurun_out/t_gemm3.log
timeout 300 python -m pytest tests/test_gpu_golden.py tests/test_gpu_permute.py -q -x --timeout 120 > gpurun_out/t_rest3.log 2>&1; echo "rest rc=$?"; tail -2 gpurun_out/t_rest3.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo "bench rc=$?"
for cg in 1 2; do for bn in 128 256; do
python - <<PY >> gpurun_out/sweep3.txt 2>&1
import torch, sys
sys.path.insert(0, '.')
from paper_2503_04771_b200 import contract
import statistics
dev = torch.device('cuda', 0)
for (M, N, K) in [(4096, 4096, 4096), (32768, 8192, 8192)]:
    a = torch.randn(M, K, device=dev).bfloat16(); b = torch.randn(K, N, device=dev).bfloat16()
    out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    f = lambda: contract('(i,k),(k,j)->(i,j)', a, b, out=out, schedule={'cta_group': $cg, 'tile_n': $bn})
    for _ in range(3): f()
    ts = []
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    print(f"cg=$cg bn=$bn {M}x{N}x{K}: {ms:.3f} ms {2*M*N*K/ms/1e9:.1f} TFLOP/s")
PY
done; done
cat gpurun_out/sweep3.txt

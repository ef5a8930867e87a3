#!/bin/bash
# ncu evidence for kernel v3 + cuBLAS comparator on the same box
python - <<'PY' > gpurun_out/cublas7.txt 2>&1
import torch, statistics
dev = torch.device('cuda', 0)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
for (M, N, K) in [(4096, 4096, 4096), (32768, 8192, 8192), (8192, 8192, 8192)]:
    a = torch.randn(M, K, device=dev).bfloat16(); b = torch.randn(K, N, device=dev).bfloat16()
    for _ in range(3): torch.matmul(a, b)
    ts = []
    for _ in range(10):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); torch.matmul(a, b); e1.record(); ts.append((e0, e1))
    torch.cuda.synchronize()
    ms = statistics.median(x.elapsed_time(y) for x, y in ts)
    print(f"cuBLAS {M}x{N}x{K}: {ms:.4f} ms {2*M*N*K/ms/1e9:.1f} TFLOP/s")
PY
cat gpurun_out/cublas7.txt
python scripts/sweep_gemm.py --shapes 4096x4096x4096,32768x8192x8192,8192x8192x8192 --cg 1,2 --bn 256 > gpurun_out/sweep7.txt 2>&1; cat gpurun_out/sweep7.txt
B="python bench.py --steps 2 --warmup 3 --no-aux --no-cpu --no-e2e"
$B > gpurun_out/plain7.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches7.csv $B > gpurun_out/ncu_launch7.log 2>&1; echo "ncu launches rc=$?"
P="python scripts/profile_kernels.py --what gemm4096,chain_gemm,perm8192,perm3d --reps 2"
$P > gpurun_out/plain7b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"tc_gemm|transpose" -c 8 -o gpurun_out/prof_r01_v3 $P > gpurun_out/ncu_full7.log 2>&1; echo "ncu full rc=$?"

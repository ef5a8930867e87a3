#!/bin/bash
P="python -c \"import torch; a=torch.randn(32768,8192,device='cuda').bfloat16(); b=torch.randn(8192,8192,device='cuda').bfloat16(); [torch.matmul(a,b) for _ in range(2)]; torch.cuda.synchronize()\""
eval $P > gpurun_out/plain12.log 2>&1 && \
eval ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__cluster_dim_x,launch__cluster_dim_y,launch__block_size,launch__shared_mem_per_block_dynamic,lts__t_bytes.sum,l1tex__m_xbar2l1tex_read_bytes.sum --clock-control none -k regex:nvjet --csv --log-file gpurun_out/cublas12.csv $P > gpurun_out/ncu12.log 2>&1; echo "ncu rc=$?"
P2="python scripts/profile_kernels.py --what chain_gemm --reps 1 --cg 2"
$P2 > gpurun_out/plain12b.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,l1tex__m_xbar2l1tex_read_bytes.sum --clock-control none -k regex:tc_gemm --csv --log-file gpurun_out/ours12.csv $P2 > gpurun_out/ncu12b.log 2>&1; echo "ncu2 rc=$?"

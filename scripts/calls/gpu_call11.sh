#!/bin/bash
python scripts/power_compare.py > gpurun_out/power11.txt 2>&1; cat gpurun_out/power11.txt
P="python -c \"import torch; a=torch.randn(32768,8192,device='cuda').bfloat16(); b=torch.randn(8192,8192,device='cuda').bfloat16(); [torch.matmul(a,b) for _ in range(2)]; torch.cuda.synchronize()\""
eval $P > gpurun_out/plain11.log 2>&1 && \
eval ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__cluster_dim_x,launch__cluster_dim_y,launch__block_size --clock-control none -k regex:gemm --csv --log-file gpurun_out/cublas11.csv $P > gpurun_out/ncu11.log 2>&1; echo "ncu rc=$?"
grep -v "^==" gpurun_out/cublas11.csv | cut -c1-300 | tail -20

#!/bin/bash
# L2 hint variants, interleaved in both orders: 48 = none, 32 = keep-only (resident slab evict_last), 0 = keep + stream evict_first, 16 = stream-only
python scripts/sweep_gemm.py --shapes 32768x8192x8192 --cg 2 --bn 512 --debug 48,32,0,16,48,32,0,16,16,0,32,48 --iters 20 > gpurun_out/c58_sweep.txt 2>&1
python scripts/sweep_gemm.py --shapes 4096x4096x4096 --cg 2 --bn 256 --debug 48,32,0,16,16,0,32,48 --iters 20 >> gpurun_out/c58_sweep.txt 2>&1
python scripts/profile_kernels.py --what chain_gemm --tile-n 512 --cg 2 --debugs 48,32,0,16 --reps 1 > /dev/null 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:tc_gemm --csv --log-file gpurun_out/c58_ncu.csv python scripts/profile_kernels.py --what chain_gemm --tile-n 512 --cg 2 --debugs 48,32,0,16 --reps 1 > gpurun_out/c58_ncu.log 2>&1
cat gpurun_out/c58_sweep.txt

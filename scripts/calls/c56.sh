#!/bin/bash
# 512-wide pair tiles: raster vs DRAM traffic (ncu) and time (events)
python scripts/sweep_gemm.py --shapes 32768x8192x8192 --cg 2 --bn 512 --raster=-16,-8,-4,-2,2,4,8,16 --iters 20 > gpurun_out/c56_sweep.txt 2>&1
python scripts/profile_kernels.py --what chain_gemm --tile-n 512 --cg 2 --rasters=-16,-8,-4,-2,2,4,8,16 --reps 2 > /dev/null 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:tc_gemm --csv --log-file gpurun_out/c56_ncu.csv python scripts/profile_kernels.py --what chain_gemm --tile-n 512 --cg 2 --rasters=-16,-8,-4,-2,2,4,8,16 --reps 2 > gpurun_out/c56_ncu.log 2>&1
cat gpurun_out/c56_sweep.txt

#!/bin/bash
for cg in 2 1; do
P="python scripts/profile_kernels.py --what chain_gemm --reps 1 --cg $cg --rasters 1,2,4,8,16,32"
$P > gpurun_out/plain8.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:tc_gemm --csv --log-file gpurun_out/raster8_cg$cg.csv $P > gpurun_out/ncu8.log 2>&1; echo "ncu rc=$?"
done

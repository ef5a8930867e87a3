#!/bin/bash
P2="python scripts/profile_kernels.py --what chain_gemm --reps 1 --cg 2 --tile-n 512 --rasters 16 --debugs 0,2"
$P2 > gpurun_out/plain16.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_write.sum,lts__t_sectors_op_write.sum --clock-control none -k regex:tc_gemm --csv --log-file gpurun_out/ours16.csv $P2 > gpurun_out/ncu16.log 2>&1; echo "ncu rc=$?"; grep -v "^==" gpurun_out/ours16.csv | cut -d, -f12- | tail -8

#!/bin/bash
P2="python scripts/profile_kernels.py --what chain_gemm --reps 1 --cg 2 --tile-n 512 --rasters -8 --debugs 4,36,0,32"
$P2 > gpurun_out/plain35.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:tc_gemm --csv --log-file gpurun_out/ours35.csv $P2 > gpurun_out/ncu35.log 2>&1; echo "ncu rc=$?"; grep -v "^==" gpurun_out/ours35.csv | cut -d, -f12- | tail -8

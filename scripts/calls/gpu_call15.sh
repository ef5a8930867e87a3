#!/bin/bash
for bn in 512 256; do
P2="python scripts/profile_kernels.py --what chain_gemm --reps 1 --cg 2 --tile-n $bn --rasters 16 --debugs 0,1,4"
$P2 > gpurun_out/plain15.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:tc_gemm --csv --log-file gpurun_out/ours15_$bn.csv $P2 > gpurun_out/ncu15.log 2>&1; echo "ncu rc=$?"; grep -v "^==" gpurun_out/ours15_$bn.csv | cut -d, -f12- | tail -9
done

#!/bin/bash
P2="python scripts/profile_kernels.py --what chain_gemm --reps 1 --cg 2 --tile-n 512 --rasters 16"
$P2 > gpurun_out/plain19.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tc_gemm -c 1 -o gpurun_out/prof19 $P2 > gpurun_out/ncu19.log 2>&1; echo "ncu rc=$?"

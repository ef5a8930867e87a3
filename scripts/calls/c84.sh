#!/bin/bash
# one full ncu capture of the chain GEMM (headline kernel), after a clean run
python scripts/profile_kernels.py --what chain_gemm --reps 1 > gpurun_out/c84_run.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:tc_gemm -c 1 -o gpurun_out/c84_chain python scripts/profile_kernels.py --what chain_gemm --reps 1 > gpurun_out/c84.log 2>&1
echo rc=$?; ls -la gpurun_out | grep c84

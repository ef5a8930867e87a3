#!/bin/bash
# one --set full capture of the headline kernel (chain GEMM, 256x512 pair tiles)
python scripts/profile_kernels.py --what chain_gemm --reps 2 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 -o gpurun_out/c63_chain_full python scripts/profile_kernels.py --what chain_gemm --reps 2 > gpurun_out/c63_ncu.log 2>&1
echo rc=$?; ls -la gpurun_out/c63_chain_full.ncu-rep

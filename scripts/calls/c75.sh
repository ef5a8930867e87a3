#!/bin/bash
python scripts/c3_probe.py && \
ncu --section LaunchStats --section Occupancy --clock-control none -k regex:nvjet -c 1 python scripts/c3_probe.py > gpurun_out/c75_launch.txt 2>&1
grep -E "nvjet|tc_gemm|Grid Size|Block Size|Cluster|Shared Memory|Registers|Waves|Threads" gpurun_out/c75_launch.txt | head -60

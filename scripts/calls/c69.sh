#!/bin/bash
python scripts/prof_8192.py 4096 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 -o gpurun_out/c69_4096 python scripts/prof_8192.py 4096 > gpurun_out/c69.log 2>&1
echo rc=$?

#!/bin/bash
python scripts/prof_ffma.py > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:simt_gemm_big -s 0 -c 1 -o gpurun_out/c70_ffma python scripts/prof_ffma.py > gpurun_out/c70.log 2>&1
echo rc=$?

#!/bin/bash
python scripts/c3_probe.py && \
ncu --set full --import-source on --clock-control none -k regex:tc_gemm -c 1 -o gpurun_out/c76_c3 python scripts/c3_probe.py > gpurun_out/c76.log 2>&1
ls -la gpurun_out/ | grep c76

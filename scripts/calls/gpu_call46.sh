#!/bin/bash
P="python scripts/simt_probe.py"
$P > gpurun_out/simt46.log 2>&1 && cat gpurun_out/simt46.log && \
ncu --set full --clock-control none --import-source on -k regex:simt_gemm_big -c 2 -o gpurun_out/prof_simt46 $P > gpurun_out/ncu46.log 2>&1; echo "ncu rc=$?"

#!/bin/bash
for rep in 1 2; do
python scripts/sweep_gemm.py --shapes 1024x1024x1024 --batch 64 --cg 2 --bn 256 --debug 0,2,4 >> gpurun_out/sweep51.txt 2>&1
python scripts/sweep_gemm.py --shapes 4096x4096x4096 --cg 2 --bn 256 --debug 0,2,4 >> gpurun_out/sweep51.txt 2>&1
done
cat gpurun_out/sweep51.txt

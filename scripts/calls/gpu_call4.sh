#!/bin/bash
S=scripts/sweep_gemm.py
python $S --cg 1,2 --bn 128,256 > gpurun_out/sweep4a.txt 2>&1
python $S --shapes 32768x8192x8192 --cg 1 --bn 256 --stages 2,3,4 >> gpurun_out/sweep4a.txt 2>&1
python $S --shapes 32768x8192x8192 --cg 2 --bn 256 --stages 3,4,5,6 >> gpurun_out/sweep4a.txt 2>&1
python $S --shapes 32768x8192x8192 --cg 1,2 --bn 256 --raster 2,4,8,16,32,64 >> gpurun_out/sweep4a.txt 2>&1
python $S --shapes 4096x4096x4096,32768x8192x8192 --cg 1,2 --bn 128,256 --debug 1 >> gpurun_out/sweep4a.txt 2>&1
python $S --shapes 8192x8192x8192,2048x2048x8192 --cg 1,2 --bn 128,256 >> gpurun_out/sweep4a.txt 2>&1
cat gpurun_out/sweep4a.txt

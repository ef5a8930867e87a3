#!/bin/bash
python scripts/sweep_gemm.py --shapes 1024x1024x1024 --batch 64 --cg 1,2 --bn 128,256 > gpurun_out/sweep49.txt 2>&1
python scripts/sweep_gemm.py --shapes 1024x1024x1024 --batch 64 --cg 2 --bn 256 --debug 1,4 >> gpurun_out/sweep49.txt 2>&1
python scripts/sweep_gemm.py --shapes 1024x1024x1024 --batch 64 --cg 2 --bn 256 --raster 1,2,4 >> gpurun_out/sweep49.txt 2>&1
cat gpurun_out/sweep49.txt

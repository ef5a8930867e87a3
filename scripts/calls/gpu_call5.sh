#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x --timeout 120 > gpurun_out/t_gemm5.log 2>&1; echo "gemm rc=$?"; tail -2 gpurun_out/t_gemm5.log
S=scripts/sweep_gemm.py
python $S --shapes 4096x4096x4096,32768x8192x8192,8192x8192x8192 --cg 1,2 --bn 128,256 > gpurun_out/sweep5.txt 2>&1
python $S --shapes 32768x8192x8192 --cg 1,2 --bn 256 --debug 1 >> gpurun_out/sweep5.txt 2>&1
python $S --shapes 32768x8192x8192 --cg 2 --bn 256 --raster 2,4,16 >> gpurun_out/sweep5.txt 2>&1
cat gpurun_out/sweep5.txt
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench5.json 2> gpurun_out/bench5.err; echo "bench rc=$?"

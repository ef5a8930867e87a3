#!/bin/bash
# full GPU suite + default bench (1 GPU)
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/c55_gpu.txt
timeout 900 python bench.py > gpurun_out/c55_bench.json 2> gpurun_out/c55_bench.err
cat gpurun_out/c55_gpu.txt; tail -3 gpurun_out/c55_bench.err; cat gpurun_out/c55_bench.json

#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_edges.py tests/test_compat.py -q -x --timeout 300 > gpurun_out/t_33.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_33.log
timeout 600 python scripts/bench_classes.py > gpurun_out/classes33.txt 2>&1; echo "rc=$?"; cat gpurun_out/classes33.txt

#!/bin/bash
timeout 600 python -m pytest tests/test_fir_gpu.py tests/test_compat.py -q --timeout 120 > gpurun_out/t_23.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/t_23.log

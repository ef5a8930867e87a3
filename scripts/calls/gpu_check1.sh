#!/bin/bash
# first GPU call: smoke pieces in isolation, then the gpu test files
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import torch;print(torch.cuda.get_device_name(0))"
timeout 120 python -m pytest tests/test_gpu_permute.py -q -x --timeout 60 > gpurun_out/t_permute.log 2>&1; echo "permute rc=$?"
timeout 300 python -m pytest tests/test_gpu_golden.py -q -x --timeout 120 > gpurun_out/t_golden.log 2>&1; echo "golden rc=$?"
timeout 120 python -m pytest tests/test_gpu_gemm.py -q -x --timeout 60 -k "fp32 or f64 or step_limit or c1" > gpurun_out/t_simt.log 2>&1; echo "simt rc=$?"
timeout 120 python -m pytest tests/test_gpu_gemm.py -q -x --timeout 60 -k "tcgen05_layouts and A_k_B_n and bfloat16 and 128-256-64" > gpurun_out/t_tc1.log 2>&1; echo "tc1 rc=$?"
timeout 300 python -m pytest tests/test_gpu_gemm.py -q --timeout 60 -k "tcgen05 or baseline or selection" > gpurun_out/t_tc.log 2>&1; echo "tc rc=$?"
tail -5 gpurun_out/t_*.log

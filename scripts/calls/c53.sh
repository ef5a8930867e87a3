#!/bin/bash
# fused K-split reduce-scatter tests + full GPU suite
timeout 600 python -m pytest tests/test_gpu_fused_ksplit.py -q -x 2>&1 | tail -30 > gpurun_out/c53_rs.txt
cat gpurun_out/c53_rs.txt

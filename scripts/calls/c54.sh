#!/bin/bash
# split-aware tile choice: new lib vs previous lib on small-output shapes; fused tests
python scripts/splitk_probe.py > gpurun_out/c54_new.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_fused_ksplit.py tests/test_gpu_gemm.py -q -x 2>&1 | tail -3 > gpurun_out/c54_tests.txt
PYTHONPATH=$PWD python scripts/rs_probe.py > gpurun_out/c54_rs.txt 2>&1
cp oldlib/libbgx.so paper_2503_04771_b200/libbgx.so
python scripts/splitk_probe.py > gpurun_out/c54_old.txt 2>&1
cat gpurun_out/c54_*.txt

#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x --timeout 300 > gpurun_out/t_44.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_44.log
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/bench44.json 2> gpurun_out/bench44.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench44.json'))
print(d['value']); print(d['aux']['c4_gemm_4096']); print(d['aux']['c3_batched_64x1024'])"

#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_permute.py -q -x --timeout 120 > gpurun_out/t_6.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_6.log
S=scripts/sweep_gemm.py
for rep in 1 2; do
python $S --shapes 4096x4096x4096,32768x8192x8192,8192x8192x8192 --cg 1,2 --bn 256 --debug 0,2 >> gpurun_out/sweep6.txt 2>&1
done
cat gpurun_out/sweep6.txt
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench6.json 2> gpurun_out/bench6.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench6.json'))
print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks'])
for k,v in (d['aux'] or {}).items(): print(k, v)
"

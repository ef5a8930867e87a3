#!/bin/bash
timeout 900 python bench.py --no-cpu > gpurun_out/bench43.json 2> gpurun_out/bench43.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench43.json'))
print(d['value'], d['e2e'], d['clocks'])"
B="python bench.py --steps 2 --warmup 3 --no-aux --no-cpu --no-e2e"
$B > gpurun_out/plain43.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches43.csv $B > gpurun_out/ncu43a.log 2>&1; echo "ncu launches rc=$?"
P="python scripts/profile_kernels.py --what chain_gemm,gemm4096,perm8192 --reps 1"
$P > gpurun_out/plain43b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"tc_gemm|transpose" -c 3 -o gpurun_out/prof_r01_v5 $P > gpurun_out/ncu43b.log 2>&1; echo "ncu full rc=$?"

#!/bin/bash
# bench + launch list + full ncu of the GEMM and the permute
python -m pytest tests/test_gpu_permute.py -q --timeout 120 > gpurun_out/t_permute.log 2>&1; echo "permute rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench rc=$?"
cat gpurun_out/bench1.json
B="python bench.py --steps 2 --warmup 3 --no-aux --no-cpu --no-e2e"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
P="python scripts/profile_kernels.py --what gemm4096,chain_gemm,perm8192 --reps 2"
$P > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"tc_gemm|transpose" -c 5 -o gpurun_out/prof_r01 $P > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
ls -la gpurun_out

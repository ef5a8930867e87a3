#!/bin/bash
# L2 eviction hints on TMA loads: A/B (debug bit 16 = no hints), interleaved; DRAM bytes under ncu
python scripts/sweep_gemm.py --shapes 32768x8192x8192 --cg 2 --bn 512 --debug 0,16,0,16,0,16 --iters 20 > gpurun_out/c57_sweep.txt 2>&1
python scripts/sweep_gemm.py --shapes 4096x4096x4096 --cg 2 --bn 256 --debug 0,16,0,16,0,16 --iters 20 >> gpurun_out/c57_sweep.txt 2>&1
python scripts/sweep_gemm.py --shapes 1024x1024x1024 --batch 64 --cg 2 --bn 256 --debug 0,16,0,16 --iters 20 >> gpurun_out/c57_sweep.txt 2>&1
python scripts/profile_kernels.py --what chain_gemm --tile-n 512 --cg 2 --debugs 0,16 --reps 2 > /dev/null 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:tc_gemm --csv --log-file gpurun_out/c57_ncu.csv python scripts/profile_kernels.py --what chain_gemm --tile-n 512 --cg 2 --debugs 0,16 --reps 2 > gpurun_out/c57_ncu.log 2>&1
cat gpurun_out/c57_sweep.txt

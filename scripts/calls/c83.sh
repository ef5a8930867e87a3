#!/bin/bash
# launch list of the bench command (run once without ncu first)
python bench.py --steps 2 --warmup 3 --no-aux --no-cpu --no-e2e > gpurun_out/c83_bench.json 2>/dev/null && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/c83_launches.csv python bench.py --steps 2 --warmup 3 --no-aux --no-cpu --no-e2e > gpurun_out/c83_ncu.log 2>&1
echo rc=$?; wc -l gpurun_out/c83_launches.csv

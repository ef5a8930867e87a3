#!/bin/bash
# launch list of the bench command (ncu only after the plain run exits 0)
python bench.py --steps 2 --warmup 3 --no-aux --no-e2e --no-cpu > gpurun_out/c62_plain.json 2> gpurun_out/c62_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c62_launches.csv python bench.py --steps 2 --warmup 3 --no-aux --no-e2e --no-cpu > gpurun_out/c62_ncu.log 2>&1
echo rc=$?; tail -3 gpurun_out/c62_launches.csv

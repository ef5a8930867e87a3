#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_host_api.py -q -s --timeout 300 > gpurun_out/t_host10.log 2>&1; echo "host tests rc=$?"; tail -5 gpurun_out/t_host10.log
timeout 900 python bench.py --no-aux --no-cpu > gpurun_out/bench10.json 2> gpurun_out/bench10.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench10.json'))
print(d['value'], d['e2e'], d['clocks'])"

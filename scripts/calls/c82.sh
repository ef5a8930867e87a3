#!/bin/bash
python -m pytest tests/test_gpu_host_api.py -x -q 2>&1 | tail -2
for i in 1 2; do python bench.py --no-aux --no-cpu --steps 8 > gpurun_out/c82_b$i.json 2>/dev/null; python -c "
import json;b=json.load(open('gpurun_out/c82_b$i.json'));print(b['value'], json.dumps(b['e2e']))"; done

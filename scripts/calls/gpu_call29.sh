#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/t_29.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_29.log
timeout 900 python bench.py > gpurun_out/bench29.json 2> gpurun_out/bench29.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench29.json'))
for k in ['value','ms_per_step','fraction_of_peak','clocks','e2e','roofline']: print(k, d.get(k))
for k,v in (d['aux'] or {}).items(): print(k, v)
"

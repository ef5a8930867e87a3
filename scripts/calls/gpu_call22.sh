#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/t_all22.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/t_all22.log
timeout 900 python bench.py > gpurun_out/bench22.json 2> gpurun_out/bench22.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench22.json'))
for k in ['value','ms_per_step','fraction_of_peak','clocks','parity','e2e','roofline']: print(k, d.get(k))
for k,v in (d['aux'] or {}).items(): print(k, v)
"

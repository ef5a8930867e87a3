#!/bin/bash
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke40.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke40.log
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/t_40.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/t_40.log
timeout 900 python bench.py > gpurun_out/bench40.json 2> gpurun_out/bench40.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench40.json'))
for k in ['value','ms_per_step','fraction_of_peak','clocks','e2e','roofline','cpu_baseline','gpu_launches']: print(k, d.get(k))
for k,v in (d['aux'] or {}).items(): print(k, v)
"

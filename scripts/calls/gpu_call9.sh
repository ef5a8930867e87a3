#!/bin/bash
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke9.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke9.log
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/t_all9.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/t_all9.log
timeout 900 python bench.py > gpurun_out/bench9.json 2> gpurun_out/bench9.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench9_ref.json 2> gpurun_out/bench9_ref.err; echo "ref rc=$?"
cat gpurun_out/bench9_ref.json

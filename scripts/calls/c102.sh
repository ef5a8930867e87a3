#!/bin/bash
# checkpoint: smoke, full GPU suite, default bench, reference arm
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c102_smoke.txt 2>&1; echo smoke rc=$? >> gpurun_out/c102_smoke.txt
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/c102_gpu.txt
timeout 900 python bench.py > gpurun_out/c102_bench.json 2> gpurun_out/c102_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/c102_ref.json 2> gpurun_out/c102_ref.err
tail -2 gpurun_out/c102_smoke.txt; cat gpurun_out/c102_gpu.txt; cut -c1-600 gpurun_out/c102_bench.json; cut -c1-400 gpurun_out/c102_ref.json

#!/bin/bash
python -m pytest tests/test_gpu_fused_ksplit.py -x -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python scripts/rs_probe.py 2>&1 | tail -4
python scripts/rs_world1_probe.py 2>&1 | head -2

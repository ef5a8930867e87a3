#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -3
python scripts/rank_slab_probe.py 2>&1 | tail -4

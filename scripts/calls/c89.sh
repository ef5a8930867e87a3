#!/bin/bash
python scripts/c1_dsl_time.py
python scripts/overhead.py 2>&1 | tail -12
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3

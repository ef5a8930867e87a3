#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/t_25.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_25.log

#!/bin/bash
timeout 600 python scripts/overhead.py > gpurun_out/overhead37.txt 2>&1; echo "rc=$?"; cat gpurun_out/overhead37.txt

#!/bin/bash
timeout 600 python scripts/bench_classes.py > gpurun_out/classes32.txt 2>&1; echo "rc=$?"; cat gpurun_out/classes32.txt

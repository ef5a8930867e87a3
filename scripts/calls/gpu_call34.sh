#!/bin/bash
python scripts/sanitize_smoke.py > gpurun_out/san_plain.log 2>&1 && \
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_smoke.py > gpurun_out/memcheck34.log 2>&1; echo "memcheck rc=$?"; tail -8 gpurun_out/memcheck34.log

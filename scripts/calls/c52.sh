#!/bin/bash
# schedule tests + full GPU suite
python -m pytest tests/test_gpu_schedule.py -q -x 2>&1 | tail -15 > gpurun_out/c52_sched.txt
python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/c52_gpu.txt
cat gpurun_out/c52_sched.txt gpurun_out/c52_gpu.txt

#!/bin/bash
BGX_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench31_2rank.json 2> gpurun_out/bench31_2rank.err; echo "2-rank rc=$?"
cat gpurun_out/bench31_2rank.json | cut -c1-600
tail -3 gpurun_out/bench31_2rank.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/bench31_ref2.json 2> gpurun_out/bench31_ref2.err; echo "ref 2-rank rc=$?"; cut -c1-200 gpurun_out/bench31_ref2.json

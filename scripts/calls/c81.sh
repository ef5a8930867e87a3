#!/bin/bash
BGX_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/c81_2rank.json 2> gpurun_out/c81_2rank.err; echo "2-rank rc=$?"
cut -c1-700 gpurun_out/c81_2rank.json; tail -3 gpurun_out/c81_2rank.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --impl reference --gpus 2 --steps 1 --warmup 3 > gpurun_out/c81_ref2.json 2> gpurun_out/c81_ref2.err; echo "ref 2-rank rc=$?"; cut -c1-300 gpurun_out/c81_ref2.json

# Round-2 evidence on one GPU: bench line, ncu launch list of a short bench
# run, and one `ncu --set full` capture of the dominant kernel (the chain GEMM)
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 --no-aux --no-cpu --no-e2e \
    > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:tc_gemm --launch-skip 3 -c 1 \
    -o /tmp/chain_full python scripts/r02/one_variant.py chain "" > gpurun_out/ncu_chain.log 2>&1
echo "ncu full rc=$?"
ncu -i /tmp/chain_full.ncu-rep --page raw --csv > gpurun_out/chain_full_raw.csv 2>&1
ncu -i /tmp/chain_full.ncu-rep --page details --csv > gpurun_out/chain_full_details.csv 2>&1
echo done

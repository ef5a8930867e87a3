#!/bin/bash
P2="python scripts/profile_kernels.py --what chain_gemm --reps 1 --cg 2 --tile-n 512 --rasters 16,-2,-4,-8,-16"
$P2 > gpurun_out/plain20.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:tc_gemm --csv --log-file gpurun_out/ours20.csv $P2 > gpurun_out/ncu20.log 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/ours20.csv')))
i=[k for k,r in enumerate(rows) if 'Metric Name' in r][0]
h=rows[i]
for r in rows[i+1:]:
    print(r[h.index('ID')], r[h.index('Metric Name')], r[h.index('Metric Value')])
PY
python - <<'PY' > gpurun_out/power20.txt 2>&1
import sys
sys.path.insert(0, 'scripts')
src = open('scripts/power_compare.py').read().split('\nfor rep in range(')[0]
exec(src)
def ours_bn(bn, raster=0, cg=2, dbg=0):
    d = _lib.BgxContractDesc()
    d.batch, d.M, d.N, d.K = 1, M, N, K
    d.a, d.b, d.out = a.data_ptr(), b.data_ptr(), out.data_ptr()
    d.a_stride[:] = [0, K, 1]; d.b_stride[:] = [0, N, 1]; d.o_stride[:] = [0, N, 1]
    d.in_dtype = d.out_dtype = _lib.BF16; d.mode = _lib.MODE_TC
    d.sched.cta_group, d.sched.tile_n, d.sched.raster = cg, bn, raster
    d.sched.reserved[0] = dbg
    sp = torch.cuda.current_stream().cuda_stream
    return lambda: lib.bgx_contract(d, sp)
for rep in range(2):
    run("cuBLAS", lambda: torch.matmul(a, b, out=out))
    for ra in (16, -4, -8):
        run(f"ours 2x512 raster{ra}", ours_bn(512, ra))
PY
cat gpurun_out/power20.txt

#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_host_api.py -q -x --timeout 120 > gpurun_out/t_17.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_17.log
P2="python scripts/profile_kernels.py --what chain_gemm --reps 1 --cg 2 --tile-n 512 --rasters 16 --debugs 0,4"
$P2 > gpurun_out/plain17.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:tc_gemm --csv --log-file gpurun_out/ours17.csv $P2 > gpurun_out/ncu17.log 2>&1; echo "ncu rc=$?"; grep -v "^==" gpurun_out/ours17.csv | cut -d, -f12- | tail -4
python - <<'PY' > gpurun_out/power17.txt 2>&1
import sys
sys.path.insert(0, 'scripts')
src = open('scripts/power_compare.py').read().split('\nfor rep in range(')[0]
exec(src)
def ours_bn(bn, raster=0, cg=2):
    d = _lib.BgxContractDesc()
    d.batch, d.M, d.N, d.K = 1, M, N, K
    d.a, d.b, d.out = a.data_ptr(), b.data_ptr(), out.data_ptr()
    d.a_stride[:] = [0, K, 1]; d.b_stride[:] = [0, N, 1]; d.o_stride[:] = [0, N, 1]
    d.in_dtype = d.out_dtype = _lib.BF16; d.mode = _lib.MODE_TC
    d.sched.cta_group, d.sched.tile_n, d.sched.raster = cg, bn, raster
    sp = torch.cuda.current_stream().cuda_stream
    return lambda: lib.bgx_contract(d, sp)
for rep in range(2):
    run("cuBLAS", lambda: torch.matmul(a, b, out=out))
    run("ours 2x512 raster16", ours_bn(512, 16))
    run("ours 2x512 raster8", ours_bn(512, 8))
PY
cat gpurun_out/power17.txt

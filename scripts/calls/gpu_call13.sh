#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x --timeout 120 > gpurun_out/t_13.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_13.log
python - <<'PY' > gpurun_out/power13.txt 2>&1
import runpy, sys
sys.argv = ['x']
PY
sed -i 's/^for rep in range(2):/for rep in range(1):/' scripts/power_compare.py
python - <<'PY' >> gpurun_out/power13.txt 2>&1
import sys, os
sys.path.insert(0, 'scripts')
src = open('scripts/power_compare.py').read().split('\nfor rep in range(1):')[0]
exec(src)
def ours_bn(bn, raster=0):
    d = _lib.BgxContractDesc()
    d.batch, d.M, d.N, d.K = 1, M, N, K
    d.a, d.b, d.out = a.data_ptr(), b.data_ptr(), out.data_ptr()
    d.a_stride[:] = [0, K, 1]; d.b_stride[:] = [0, N, 1]; d.o_stride[:] = [0, N, 1]
    d.in_dtype = d.out_dtype = _lib.BF16; d.mode = _lib.MODE_TC
    d.sched.cta_group, d.sched.tile_n, d.sched.raster = 2, bn, raster
    sp = torch.cuda.current_stream().cuda_stream
    return lambda: lib.bgx_contract(d, sp)
for rep in range(2):
    run("cuBLAS", lambda: torch.matmul(a, b, out=out))
    run("ours 2x256", ours_bn(256))
    run("ours 2x512", ours_bn(512))
    run("ours 2x512 raster4", ours_bn(512, 4))
    run("ours 2x512 raster16", ours_bn(512, 16))
PY
cat gpurun_out/power13.txt
P2="python scripts/profile_kernels.py --what chain_gemm --reps 1 --cg 2 --tile-n 512 --rasters 2,4,8,16"
$P2 > gpurun_out/plain13.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum --clock-control none -k regex:tc_gemm --csv --log-file gpurun_out/ours13.csv $P2 > gpurun_out/ncu13.log 2>&1; echo "ncu rc=$?"

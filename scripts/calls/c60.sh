#!/bin/bash
# instruction / traffic counters: ours (256, 512) vs cuBLAS at 4096^3
python scripts/prof_8192.py 4096 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,smsp__inst_executed_op_shared_st.sum,smsp__inst_executed_op_shared_ld.sum,lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__warps_active.avg.per_cycle_active,smsp__inst_executed_pipe_uniform.sum --clock-control none --csv --log-file gpurun_out/c60_ncu.csv python scripts/prof_8192.py 4096 > gpurun_out/c60.log 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/c60_ncu.csv')))
hdr=None; data={}
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); data.setdefault(d['ID'],(d['Kernel Name'][:50],{}))[1][d['Metric Name']]=d['Metric Value']
for k in sorted(data,key=int):
    if 'copy' in data[k][0]: continue
    print(k, data[k][0]); print('   ', data[k][1])
PY

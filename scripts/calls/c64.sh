#!/bin/bash
python scripts/prof_batched.py > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/c64_ncu.csv python scripts/prof_batched.py > gpurun_out/c64.log 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/c64_ncu.csv')))
hdr=None; data={}
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); data.setdefault(d['ID'],(d['Kernel Name'][:50],{}))[1][d['Metric Name']]=d['Metric Value']
for k in sorted(data,key=int):
    if 'distribution' in data[k][0] or 'copy' in data[k][0]: continue
    print(k, data[k][0]); print('   ', data[k][1])
PY

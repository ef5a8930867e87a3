#!/bin/bash
python scripts/prof_8192.py > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/c59_ncu.csv python scripts/prof_8192.py > gpurun_out/c59.log 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/c59_ncu.csv')))
hdr=None; data={}
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); data.setdefault(d['ID'],(d['Kernel Name'][:60],{}))[1][d['Metric Name']]=d['Metric Value']
for k in sorted(data,key=int): print(k, data[k][0], data[k][1])
PY

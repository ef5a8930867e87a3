#!/bin/bash
python scripts/c3_probe.py && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,smsp__inst_executed.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/c74_ncu.csv python scripts/c3_probe.py > gpurun_out/c74.log 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/c74_ncu.csv')))
hdr=None; data={}; names={}
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); data.setdefault(d['ID'],{})[d['Metric Name']]=d['Metric Value']; names[d['ID']]=d['Kernel Name'][:60]
for k in sorted(data,key=int):
    m=data[k]; print(k, names[k][:40], *[f"{x.split('__')[1][:22]}={m[x]}" for x in sorted(m)])
PY

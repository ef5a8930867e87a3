#!/bin/bash
python scripts/profile_kernels.py --what perm8192,perm3d --reps 2 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum --clock-control none -k regex:transpose --csv --log-file gpurun_out/c103_ncu.csv python scripts/profile_kernels.py --what perm8192,perm3d --reps 2 > gpurun_out/c103.log 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/c103_ncu.csv')))
hdr=None; data={}; names={}
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); data.setdefault(d['ID'],{})[d['Metric Name']]=d['Metric Value']+d['Metric Unit']; names[d['ID']]=d['Kernel Name'][:40]
for k in sorted(data,key=int): print(k, names[k], data[k])
PY

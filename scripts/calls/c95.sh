#!/bin/bash
python scripts/profile_kernels.py --what chain_gemm --debugs 0,32,64 --reps 1 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:tc_gemm --csv --log-file gpurun_out/c95_ncu.csv python scripts/profile_kernels.py --what chain_gemm --debugs 0,32,64 --reps 1 > gpurun_out/c95.log 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/c95_ncu.csv')))
hdr=None; data={}
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); data.setdefault(d['ID'],{})[d['Metric Name']]=d['Metric Value']
for k,lab in zip(sorted(data,key=int),["fwd","rev-odd-M","rev-odd-wave"]):
    m=data[k]; print(lab, *[f"{x.split('__')[1][:14]}={v}" for x,v in sorted(m.items())])
PY
AB_SCHED="reserved=64" true

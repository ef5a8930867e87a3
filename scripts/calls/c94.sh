#!/bin/bash
R="-3,-5,-6,-7,-8,-10,-12,12"
python scripts/profile_kernels.py --what chain_gemm --rasters=$R --reps 1 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:tc_gemm --csv --log-file gpurun_out/c94_ncu.csv python scripts/profile_kernels.py --what chain_gemm --rasters=$R --reps 1 > gpurun_out/c94.log 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/c94_ncu.csv')))
hdr=None; data={}
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); data.setdefault(d['ID'],{})[d['Metric Name']]=(d['Metric Value'],d['Metric Unit'])
for k,lab in zip(sorted(data,key=int),"-3,-5,-6,-7,-8,-10,-12,12".split(",")):
    m=data[k]; print("raster",lab, *[f"{x.split('__')[1][:14]}={v[0]}{v[1]}" for x,v in sorted(m.items())])
PY

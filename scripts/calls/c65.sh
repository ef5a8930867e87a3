#!/bin/bash
python scripts/prof_fabric.py > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,lts__t_sectors.sum,lts__t_sectors_srcunit_tex.sum,lts__t_sectors_srcunit_ltcfabric.sum,dram__bytes_read.sum --clock-control none -k regex:tc_gemm --csv --log-file gpurun_out/c65_ncu.csv python scripts/prof_fabric.py > gpurun_out/c65.log 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/c65_ncu.csv')))
hdr=None; data={}
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); data.setdefault(d['ID'],{})[d['Metric Name']]=d['Metric Value']
labels=[f"{c}:{d}" for c in ("batched","4096","chain") for d in (0,256,512)]
for k,lab in zip(sorted(data,key=int),labels):
    m=data[k]
    print(lab, "us", float(m['gpu__time_duration.sum'])/1e3, "MHz", round(float(m['sm__cycles_elapsed.avg.per_second'])/1e6), "L2 sectors", m['lts__t_sectors.sum'], "tex", m['lts__t_sectors_srcunit_tex.sum'], "fabric", m['lts__t_sectors_srcunit_ltcfabric.sum'], "dram_rd", m['dram__bytes_read.sum'])
PY

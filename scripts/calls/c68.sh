#!/bin/bash
timeout 120 python scripts/prof_die.py 2>&1 | tail -4
timeout 120 python scripts/prof_die.py > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,lts__t_sectors_srcunit_tex.sum,lts__t_sectors_srcunit_ltcfabric.sum,dram__bytes_read.sum --clock-control none -k regex:tc_gemm --csv --log-file gpurun_out/c68_ncu.csv python scripts/prof_die.py > gpurun_out/c68.log 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/c68_ncu.csv')))
hdr=None; data={}
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); data.setdefault(d['ID'],{})[d['Metric Name']]=d['Metric Value']
labels=[f"{c} {m}" for c in ("chain","batched","8192^3") for m in ("static","die-affine")]
for k,lab in zip(sorted(data,key=int),labels):
    m=data[k]
    print(f"{lab:20s} {float(m['gpu__time_duration.sum'])/1e3:8.1f} us {float(m['sm__cycles_elapsed.avg.per_second'])/1e6:6.0f} MHz tex {int(m['lts__t_sectors_srcunit_tex.sum'])*32/1e9:.2f} GB fabric {int(m['lts__t_sectors_srcunit_ltcfabric.sum'])*32/1e9:.2f} GB dram_rd {int(m['dram__bytes_read.sum'])/1e9:.2f} GB")
PY

#!/bin/bash
python scripts/c3_probe.py "" "tile_n=512,cta_group=2" && \
ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,lts__t_sectors_op_read.sum,smsp__inst_executed.sum,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"nvjet|tc_gemm" --csv --log-file gpurun_out/c77_ncu.csv python scripts/c3_probe.py "" "tile_n=512,cta_group=2" > gpurun_out/c77.log 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/c77_ncu.csv')))
hdr=None; data={}; names={}
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); data.setdefault(d['ID'],{})[d['Metric Name']]=d['Metric Value']; names[d['ID']]=d['Kernel Name'][:40]
for k in sorted(data,key=int):
    m=data[k]; print(k, names[k], *[f"{x.split('__')[1][:26]}={m[x]}" for x in sorted(m)])
PY

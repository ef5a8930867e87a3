#!/bin/bash
python scripts/c3_probe.py "" "tile_n=512,cta_group=2" && \
ncu --metrics gpu__time_duration.sum,l1tex__m_xbar2l1tex_read_sectors_mem_global_op_tma_ld.sum,lts__t_sectors_srcunit_ltcfabric.sum,lts__t_requests_srcunit_ltcfabric.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,dram__bytes_read.sum --clock-control none -k regex:"nvjet|tc_gemm" --csv --log-file gpurun_out/c79_ncu.csv python scripts/c3_probe.py "" "tile_n=512,cta_group=2" > gpurun_out/c79.log 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/c79_ncu.csv')))
hdr=None; data={}; names={}
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); data.setdefault(d['ID'],{})[d['Metric Name']]=d['Metric Value']; names[d['ID']]=d['Kernel Name'][:40]
for k in sorted(data,key=int):
    m=data[k]; print(k, names[k], *[f"{x[:40]}={m[x]}" for x in sorted(m)])
PY

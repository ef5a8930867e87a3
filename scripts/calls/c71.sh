#!/bin/bash
python scripts/profile_kernels.py --what chain_gemm --debugs 0,16 --reps 1 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct --clock-control none -k regex:tc_gemm --csv --log-file gpurun_out/c71_ncu.csv python scripts/profile_kernels.py --what chain_gemm --debugs 0,16,0,16 --reps 1 > gpurun_out/c71.log 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/c71_ncu.csv')))
hdr=None; data={}
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); data.setdefault(d['ID'],{})[d['Metric Name']]=d['Metric Value']
for k,lab in zip(sorted(data,key=int),["evict_first","normal","evict_first","normal"]):
    m=data[k]; print(lab, m['gpu__time_duration.sum'], m['dram__bytes_read.sum'], m['dram__bytes_write.sum'], m['lts__t_sector_hit_rate.pct'], m['sm__cycles_elapsed.avg.per_second'][:6])
PY
python scripts/ab_lib.py paper_2503_04771_b200/libbgx.so oldlib/libbgx.so c5_chain_gemm,c4_4096 2>&1 | tail -12

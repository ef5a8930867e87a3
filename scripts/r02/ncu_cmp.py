"""Side-by-side of selected raw ncu metrics from several --page raw CSVs."""
import csv
import re
import sys

PATS = sys.argv[2].split("|") if len(sys.argv) > 2 and sys.argv[1] == "-m" else None
files = sys.argv[3:] if PATS else sys.argv[1:]
DEFAULT = [r"^gpu__time_duration.sum$", r"^sm__cycles_elapsed.avg.per_second$",
           r"sm__pipe_tensor.*hmma.*pct|sm__pipe_tensor_subpipe_hmma.*pct|tensor.*active.*pct",
           r"^lts__t_sectors.sum$", r"^lts__t_requests.sum$", r"lts__t_sectors_srcunit_tex.sum$",
           r"^lts__throughput.avg.pct_of_peak_sustained_elapsed$", r"^dram__bytes_read.sum$",
           r"^dram__bytes_write.sum$", r"lts__t_sectors_srcunit_ltcfabric.sum$",
           r"^l1tex__m_xbar2l1tex_read_sectors.sum$", r"^lts__d_sectors_fill",
           r"^smsp__inst_executed.sum$", r"lts__average_t_sector", r"^lts__t_sector_hit_rate.pct$",
           r"^sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed$",
           r"^sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct", r"^lts__t_sectors_srcunit_tex_op_write.sum$",
           r"^lts__t_sectors_srcunit_tex_op_read.sum$", r"^sm__throughput.avg.pct", r"^lts__t_requests_srcunit_tex.sum$"]
pats = [re.compile(p) for p in (PATS or DEFAULT)]
tables = []
for f in files:
    rows = list(csv.reader(open(f)))
    hdr_i = next(i for i, r in enumerate(rows) if "ID" in r or "Kernel Name" in r)
    hdr, units, vals = rows[hdr_i], rows[hdr_i + 1], rows[hdr_i + 2]
    tables.append({h: (v, u) for h, u, v in zip(hdr, units, vals)})
keys = [k for k in tables[0] if any(p.search(k) for p in pats)]
print("metric".ljust(70), *[f.split("/")[-1][:28].ljust(28) for f in files])
for k in keys:
    print(k[:70].ljust(70), *[(t.get(k, ("?", ""))[0] + " " + t.get(k, ("", ""))[1])[:28].ljust(28) for t in tables])

"""Summarise gpurun_out/kind_<config>.csv: last execution of each mode, per kernel launch."""
import csv
import sys
from collections import defaultdict

for path in sys.argv[1:]:
    rows = [r for r in csv.reader(open(path)) if r and r[0].startswith('"') is False]
    lines = [l for l in open(path) if l.startswith('"')]
    rd = list(csv.reader(lines))
    h = rd[0]
    data = rd[1:]
    by = defaultdict(dict)
    names = {}
    for r in data:
        i = int(r[h.index("ID")])
        by[i][r[h.index("Metric Name")]] = r[h.index("Metric Value")]
        names[i] = r[h.index("Kernel Name")]
    print("==", path)
    for i in sorted(by):
        m = by[i]
        print(f"{i:3d} {names[i][:40]:40s} {float(m['gpu__time_duration.sum'])/1e3:8.1f}us inst {float(m['smsp__inst_executed.sum'])/1e6:7.1f}M l1pipe {m['l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_active']}% issue {m['smsp__issue_active.avg.pct_of_peak_sustained_active']}% L2hit {m['lts__t_sector_hit_rate.pct']}% dram {float(m['dram__bytes_read.sum'])/1e6:.0f}MB occ {m.get('sm__warps_active.avg.pct_of_peak_sustained_active', '-')}%")

#!/usr/bin/env python
"""Print a per-kernel table from an ncu --csv launch list (metrics: duration, dram r/w,
fp64 pipe, instructions): python tools/launch_breakdown.py gpurun_out/x.csv [--last N]"""
import collections
import csv
import sys

path = sys.argv[1]
last = int(sys.argv[sys.argv.index("--last") + 1]) if "--last" in sys.argv else 1000
rows = list(csv.reader(open(path)))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d, names = collections.defaultdict(dict), {}
for r in rows[hdr + 1:]:
    d[r[ii]][r[mi]] = r[vi]
    names[r[ii]] = r[ki].split("(")[0][:48]
tot = 0.0
out = []
for k in sorted(d, key=int)[-last:]:
    m = d[k]
    t = float(m.get("gpu__time_duration.sum", "0").replace(",", ""))
    tot += t
    out.append((names[k], t, m))
for n, t, m in out:
    print(f"{n:48s} {t / 1e3:9.1f} us {100 * t / tot:5.1f}%  rd {m.get('dram__bytes_read.sum', '-'):>12s} "
          f"wr {m.get('dram__bytes_write.sum', '-'):>12s} fp64% {m.get('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', '-'):>6s}")
print(f"total {tot / 1e3:.1f} us")

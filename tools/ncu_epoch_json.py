#!/usr/bin/env python
"""Per-kernel table of one epoch from an ncu --csv launch list (metrics: duration, dram r/w,
fp64 pipe) of tools/epoch_run.py, recorded for bench.py's roofline.ncu_epoch:
    python tools/ncu_epoch_json.py gpurun_out/x.csv WORKLOAD --last K
K = the number of kernel launches of one epoch (the last K of the list are taken).
Updates profiles/r2/launch_shares.json."""
import collections
import csv
import json
import os
import sys

path, workload = sys.argv[1], sys.argv[2]
last = int(sys.argv[sys.argv.index("--last") + 1])
rows = list(csv.reader(open(path)))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, ii, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID"), \
    h.index("Metric Unit")
d, names = collections.defaultdict(dict), {}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6,
         "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9, "%": 1}
for r in rows[hdr + 1:]:
    d[r[ii]][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
    names[r[ii]] = r[ki].split("(")[0].replace("void ", "").replace("pmf::", "").replace("pln::", "")
ids = sorted(d, key=int)[-last:]
ks = []
for i in ids:
    m = d[i]
    ks.append({"name": names[i], "us": 1e6 * m.get("gpu__time_duration.sum", 0.0),
               "dram_bytes": m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0),
               "fp64_pipe_pct": m.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")})
tot = sum(k["us"] for k in ks)
for k in ks:
    k["share"] = k["us"] / tot if tot else None
rec = {"kernels": ks, "us_per_epoch_ncu": tot, "dram_bytes_per_epoch": sum(k["dram_bytes"] for k in ks),
       "source": os.path.relpath(path), "note": "ncu --clock-control none, cold cache, serialised launches"}
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "r2", "launch_shares.json")
allr = json.load(open(out)) if os.path.exists(out) else {}
allr[workload] = rec
json.dump(allr, open(out, "w"), indent=1)
print(json.dumps(rec, indent=1))

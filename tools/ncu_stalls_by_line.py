#!/usr/bin/env python
"""Stall-reason breakdown per CUDA source line for one kernel of an ncu report:
python tools/ncu_stalls_by_line.py rep.ncu-rep KERNEL_SUBSTR [FILE_SUBSTR] [--top 25]"""
import collections
import csv
import io
import subprocess
import sys

rep, ks = sys.argv[1], sys.argv[2]
fs = sys.argv[3] if len(sys.argv) > 3 and not sys.argv[3].startswith("--") else ""
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 25
out = subprocess.run(["ncu", "-i", rep, "--csv", "--page", "source", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file, cur_fn, hdr, line = None, None, None, None
agg = collections.defaultdict(collections.Counter)
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        cur_fn = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or ks not in (cur_fn or "") or fs not in (cur_file or ""):
        continue
    if r[0]:
        key = (cur_file, int(r[0]), r[1].strip()[:60])
        for j, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h and j < len(r) and r[j]:
                try:
                    agg[key][h[6:]] += int(r[j])
                except ValueError:
                    pass
tot = sum(sum(c.values()) for c in agg.values()) or 1
for k, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:top]:
    s = sum(c.values())
    parts = ", ".join(f"{n} {100 * v / s:.0f}%" for n, v in c.most_common(3))
    print(f"{100 * s / tot:5.1f}%  {k[0]}:{k[1]:4d} {k[2]:60s} | {parts}")

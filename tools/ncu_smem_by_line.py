#!/usr/bin/env python
"""Shared-memory wavefronts (total and excessive = bank-conflict replays) per CUDA source line
for one kernel of an ncu --set full report compiled with -lineinfo:
python tools/ncu_smem_by_line.py rep.ncu-rep KERNEL_SUBSTR [--top 25]"""
import collections
import csv
import io
import subprocess
import sys

rep, ks = sys.argv[1], sys.argv[2]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 25
out = subprocess.run(["ncu", "-i", rep, "--csv", "--page", "source", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file, cur_fn, hdr = None, None, None
agg = collections.defaultdict(lambda: [0, 0, 0])
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
    if hdr is None or ks not in (cur_fn or "") or not r[0]:
        continue
    key = (cur_file, int(r[0]), r[1].strip()[:70])
    for j, name in enumerate(("L1 Wavefronts Shared", "L1 Wavefronts Shared Excessive", "L1 Wavefronts Shared Ideal")):
        i = hdr.index(name)
        try:
            agg[key][j] += int(float(r[i] or 0))
        except ValueError:
            pass
tot = sum(v[0] for v in agg.values()) or 1
exc = sum(v[1] for v in agg.values())
print(f"shared wavefronts {tot}, excessive {exc} ({100 * exc / tot:.1f} %)")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * v[0] / tot:5.1f}%  exc {v[1]:9d} ideal {v[2]:9d}  {k[0]}:{k[1]:4d} {k[2]}")

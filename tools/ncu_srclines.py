#!/usr/bin/env python
"""Executed warp instructions and stall samples per CUDA source line for one kernel of an
ncu report (compiled with -lineinfo): python tools/ncu_lines.py rep.ncu-rep KERNEL_SUBSTR [--top 30]"""
import csv
import io
import subprocess
import sys

rep, ksub = sys.argv[1], sys.argv[2]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
out = subprocess.run(["ncu", "-i", rep, "--csv", "--page", "source", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file, cur_fn, res = None, None, {}
hdr = None
line = None
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
    if hdr is None or ksub not in (cur_fn or ""):
        continue
    ie = hdr.index("Instructions Executed")
    ws = hdr.index("Warp Stall Sampling (All Samples)")
    if r[0]:
        line = (cur_file, int(r[0]), r[1].strip()[:70])
        v = res.setdefault(line, [0, 0])
        try:
            v[0] += int(r[ie] or 0)
            v[1] += int(r[ws] or 0)
        except ValueError:
            pass
tot_i = sum(v[0] for v in res.values()) or 1
tot_s = sum(v[1] for v in res.values()) or 1
print(f"total warp instr {tot_i:.3e}, stall samples {tot_s}")
for k, v in sorted(res.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * v[0] / tot_i:5.1f}% inst {100 * v[1] / tot_s:5.1f}% stall  {k[0]}:{k[1]}  {k[2]}")

#!/usr/bin/env python
"""Per-source-line warp-stall samples of the kernels in an ncu report (read here):
    python tools/ncu_lines.py REPORT [--kernel SUBSTR] [--top 30]
Uses the 'cuda,sass' correlation view (-lineinfo): rows with a line number carry the
line's aggregated samples."""
import argparse
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--kernel", default="")
ap.add_argument("--top", type=int, default=30)
a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.rep, "--csv", "--page", "source", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
acc, seen, fname, func = {}, set(), "", ""
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        func = r[1]
        continue
    if r[0] == "Line No" or not r[0] or a.kernel not in func:
        continue
    key = (func, fname, r[0])
    if key in seen:          # each kernel's view can be printed twice
        continue
    seen.add(key)
    try:
        acc[(func[:60], fname, int(r[0]), r[1].strip()[:90])] = int(r[4])
    except (ValueError, IndexError):
        pass
funcs = sorted({k[0] for k in acc})
for f in funcs:
    items = [(v, k) for k, v in acc.items() if k[0] == f]
    tot = sum(v for v, _ in items) or 1
    print(f"== {f}  (samples {tot})")
    for v, k in sorted(items, reverse=True)[:a.top]:
        print(f"  {100 * v / tot:5.1f}%  {k[1]}:{k[2]:<5d} {k[3]}")

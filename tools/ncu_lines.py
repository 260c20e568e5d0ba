#!/usr/bin/env python
"""Aggregate an ncu report's sampled stalls and executed instructions per CUDA
source line (needs -lineinfo): python tools/ncu_lines.py rep [--ranges a-b:name,...]"""
import argparse
import collections
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--file", default="kernels_resident.cu")
    ap.add_argument("--ranges", default="")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--csv", "--page", "source", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur = None
    samp, inst = collections.Counter(), collections.Counter()
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0].isdigit():
            key = (cur, int(r[0]), r[1].strip()[:70])
            try:
                samp[key] += int(r[4] or 0)
                inst[key] += int(r[7] or 0)
            except (ValueError, IndexError):
                pass
    ts, ti = sum(samp.values()) or 1, sum(inst.values()) or 1
    print(f"samples {ts}  warp-instructions {ti}")
    if a.ranges:
        # attribute inlined helper lines (other files) to the kernel line that called them: not
        # possible from this view, so ranges cover kernel-file lines only
        for spec in a.ranges.split(","):
            rng, name = spec.split(":")
            lo, hi = map(int, rng.split("-"))
            s = sum(v for k, v in samp.items() if k[0] == a.file and lo <= k[1] <= hi)
            i = sum(v for k, v in inst.items() if k[0] == a.file and lo <= k[1] <= hi)
            print(f"  {name:10s} lines {lo}-{hi}: samples {100 * s / ts:5.1f}%  instr {100 * i / ti:5.1f}%")
        other = sum(v for k, v in samp.items() if k[0] != a.file)
        print(f"  other files (inlined helpers): samples {100 * other / ts:5.1f}%")
    for k, v in samp.most_common(a.top):
        print(f"{100 * v / ts:5.1f}% {100 * inst[k] / ti:5.1f}%i {k[0]}:{k[1]} {k[2]}")


if __name__ == "__main__":
    main()

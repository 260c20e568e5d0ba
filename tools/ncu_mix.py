#!/usr/bin/env python
"""Executed-instruction mix by opcode (warp-level counts) of each kernel in an ncu report:
python tools/ncu_mix.py rep.ncu-rep [--top 20]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 20
out = subprocess.run(["ncu", "-i", rep, "--csv", "--page", "source", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
i = 0
seen = set()
while i < len(rows):
    if rows[i] and rows[i][0] == "Kernel Name":
        name = rows[i][1]
        hdr = rows[i + 1]
        si, ei = hdr.index("Source"), hdr.index("Instructions Executed")
        j = i + 2
        mix = collections.Counter()
        while j < len(rows) and not (rows[j] and rows[j][0] == "Kernel Name"):
            r = rows[j]
            if len(r) > ei and r[ei]:
                toks = r[si].split()
                if toks:
                    op = toks[1] if toks[0].startswith("@") else toks[0]
                    mix[op.split(".")[0]] += int(r[ei])
            j += 1
        key = (name, sum(mix.values()))
        if key not in seen:
            seen.add(key)
            tot = sum(mix.values())
            print(f"{name[:70]}  total warp instr {tot:.3e}")
            for op, v in mix.most_common(top):
                print(f"   {op:10s} {v:12d} {100 * v / tot:5.1f}%")
        i = j
    else:
        i += 1

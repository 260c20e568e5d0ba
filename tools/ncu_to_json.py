#!/usr/bin/env python
"""Record the ncu numbers bench.py reports (traffic, FP64-pipe use) for a kernel:
    python tools/ncu_to_json.py gpurun_out/prof.ncu-rep --name "k_resident_epoch<double, 1, 1>" \
        --source profiles/r1_resident_ncu.txt
Writes/updates profiles/kernel_metrics.json."""
import argparse
import csv
import io
import json
import os
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--name", required=True)
ap.add_argument("--source", default=None)
ap.add_argument("--idx", type=int, default=0, help="which profiled launch in the report")
a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.rep, "--csv", "--page", "raw"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h, u, v = r[0], r[1], r[2 + a.idx]
d = dict(zip(h, v))
unit = dict(zip(h, u))


def num(k):
    x = float(d[k].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
             "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}.get(unit.get(k, ""), 1)
    return x * scale


m = {"dram_bytes": num("dram__bytes_read.sum") + num("dram__bytes_write.sum"),
     "dram_read": num("dram__bytes_read.sum"), "dram_write": num("dram__bytes_write.sum"),
     "duration_s": num("gpu__time_duration.sum"),
     "fp64_pipe_pct": float(d["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]),
     "smem_wavefronts_pct": float(d["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"]),
     "sm_clock_hz": num("sm__cycles_elapsed.avg.per_second") * (1e9 if unit.get("sm__cycles_elapsed.avg.per_second") == "Ghz" else 1),
     "source": a.source or a.rep}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "kernel_metrics.json")
allm = json.load(open(path)) if os.path.exists(path) else {}
allm[a.name] = m
json.dump(allm, open(path, "w"), indent=1)
print(json.dumps({a.name: m}, indent=1))

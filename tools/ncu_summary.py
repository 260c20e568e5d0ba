#!/usr/bin/env python
"""Summarise an ncu report (read here, no GPU): key throughput metrics, stall
reasons, and the hottest SASS instructions.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--top 12] [--out profiles/x.txt]
"""
import argparse
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "sm clock"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC"),
    ("smsp__sass_inst_executed_op_local_ld.sum", "local ld (spills)"),
    ("smsp__sass_inst_executed_op_local_st.sum", "local st (spills)"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, "--csv", *args], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=12)
    ap.add_argument("--out", default=None)
    ap.add_argument("--idx", type=int, default=0, help="which profiled launch in the report")
    a = ap.parse_args()
    lines = []
    p = lines.append
    raw = ncu_csv(a.rep, "--page", "raw")
    h, units, vals = raw[0], raw[1], raw[2 + a.idx]
    d = dict(zip(h, vals))
    u = dict(zip(h, units))
    p(f"report: {a.rep}")
    p(f"kernel: {d.get('Kernel Name', '?')}")
    for k, name in KEYS:
        if k in d:
            p(f"  {name:22s} {d[k]} {u.get(k, '')}")
    st = []
    for k in h:
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(d[k]), k.replace("smsp__average_warps_issue_stalled_", "").replace(
                    "_per_issue_active.ratio", "")))
            except ValueError:
                pass
    st.sort(reverse=True)
    p("  stall reasons (warp-cycles per issued instruction):")
    for v, k in st[:10]:
        p(f"    {k:24s} {v:.3f}")
    allrows = ncu_csv(a.rep, "--page", "source", "--print-source", "sass")
    starts = [i for i, r in enumerate(allrows) if r and r[0] == "Kernel Name"]
    # newer ncu prints every kernel's SASS section twice: keep one section per kernel name change
    firsts = [i for j, i in enumerate(starts) if j == 0 or allrows[i][1] != allrows[starts[j - 1]][1]]
    ends = {i: (starts[starts.index(i) + 1] if starts.index(i) + 1 < len(starts) else None) for i in firsts}
    rows = allrows[firsts[a.idx]:ends[firsts[a.idx]]] if a.idx < len(firsts) else []
    if len(rows) > 2:
        hh = rows[1]
        si, ni = hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)")
        data = [r for r in rows[2:] if len(r) > ni]
        tot = sum(int(r[ni] or 0) for r in data) or 1
        ops = collections.Counter()
        for r in data:
            toks = r[si].split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") else toks[0]
            ops[op.split(".")[0]] += int(r[ni] or 0)
        p(f"  sampled stalls by opcode (total {tot}):")
        for op, v in ops.most_common(10):
            p(f"    {op:10s} {100 * v / tot:5.1f}%")
        idx = sorted(range(len(data)), key=lambda i: -int(data[i][ni] or 0))[:a.top]
        p("  hottest instructions:")
        for i in idx:
            prev = data[i - 1][si].strip() if i else ""
            p(f"    {100 * int(data[i][ni]) / tot:5.1f}%  #{i:6d}  {data[i][si].strip()[:60]:60s} <- {prev[:50]}")
        p(f"  SASS instructions in kernel: {len(data)}")
    txt = "\n".join(lines)
    print(txt)
    if a.out:
        with open(a.out, "w") as f:
            f.write(txt + "\n")


if __name__ == "__main__":
    main()

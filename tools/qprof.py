#!/usr/bin/env python
"""Phase breakdown of the C4 K2 kernel (k_q_mid) from a -DPMF_QPROF build:
    PMF_NVCC_EXTRA=-DPMF_QPROF python -m paper_2412_07240_b200.build --force
    python tools/qprof.py [epochs]"""
import ctypes as C
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
E = sys.argv[1] if len(sys.argv) > 1 else "3"
from paper_2412_07240_b200 import pmf  # noqa: E402

lib = pmf.load_library()
lib.pmf_debug_counters.restype = C.c_int
lib.pmf_debug_counters.argtypes = [C.POINTER(C.c_double), C.c_int, C.c_int]
import runpy  # noqa: E402
sys.argv = ["epoch_run.py", "C4", E]
runpy.run_path(os.path.join(ROOT, "tools", "epoch_run.py"), run_name="__main__")
buf = (C.c_double * 16)()
lib.pmf_debug_counters(buf, 16, 1)
v = list(buf)
for title, idx, cnt, names in (
        ("K2 k_q_mid, per item", 0, 5, ["tables (Psi + regrid taps)", "wait for the plane", "split regrid + F2",
                                        "F2..F3 end", "I2 + refill"]),
        ("K3 k_q_inv, per plane", 11, 15, ["wait TMA plane", "inverse axis 0", "inverse axis 1",
                                          "likelihood + store + moments"])):
    n_ = v[cnt] or 1
    print(f"{title}: {n_:.0f} units; cycles per unit (thread 0 of each CTA):")
    for i, nm in enumerate(names):
        print(f"  {nm:30s} {v[idx + i] / n_:10.0f}")

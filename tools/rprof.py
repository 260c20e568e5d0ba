#!/usr/bin/env python
"""Phase breakdown of the C5 resident epoch kernel from a -DPMF_QPROF build:
    PMF_NVCC_EXTRA=-DPMF_QPROF python -m paper_2412_07240_b200.build
    python tools/rprof.py [epochs] [batch]"""
import ctypes as C
import os
import runpy
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
E = sys.argv[1] if len(sys.argv) > 1 else "3"
from paper_2412_07240_b200 import pmf  # noqa: E402

lib = pmf.load_library()
lib.pmf_debug_counters.restype = C.c_int
lib.pmf_debug_counters.argtypes = [C.POINTER(C.c_double), C.c_int, C.c_int]
sys.argv = ["epoch_run.py", "C5", E]
runpy.run_path(os.path.join(ROOT, "tools", "epoch_run.py"), run_name="__main__")
buf = (C.c_double * 28)()
lib.pmf_debug_counters(buf, 28, 1)
v = list(buf)[16:]
n = v[6] or 1
names = ["wait staged filter", "P1 load (+ regrid gather)", "P1 FFT axis 1 + unpack", "P2 rows: FFT, Psi, inverse",
         "P3 inverse axis 1 (first half)", "P3 dft16 + likelihood + store + sums"]
print(f"resident kernel: {n:.0f} filter-epochs; cycles per filter (thread 0 of each CTA):")
for i, nm in enumerate(names):
    print(f"  {nm:40s} {v[i] / n:10.0f}")
print(f"    of which: stage next + twiddle + dft16 {v[7] / n:10.0f}; likelihood + stores {v[8] / n:10.0f}; "
      f"sums + barrier {(v[5] - v[7] - v[8]) / n:10.0f}")

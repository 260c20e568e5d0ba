#!/usr/bin/env python
"""Write the full-size oracle fixtures the GPU parity tests compare against (test
infrastructure: calls only oracle/ and workloads/, never the CUDA path):

    python tools/make_golden.py C4 2 8192      # 96^4, epochs 0..2, 8192 sampled weights per epoch
    python tools/make_golden.py C3 50 2048     # 128^3, all 50 epochs

tests/golden/<cfg>_full_T<T>.npz holds, per epoch k: the moments, log normaliser and grid
of O.run_filter (R15 epoch order), the posterior weights (library layout, axis 0 fastest)
at seeded sample positions (plus the position of the peak) and the peak |w|; and the final
(regridded) weights at the same positions with the final grid."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import pmf_oracle as O  # noqa: E402
from workloads import make_config, simulate  # noqa: E402

cid, T, ns = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
cfg = make_config(cid)
zs = simulate(cfg, T=T)["z"]
t0 = time.time()
rec = O.run_filter(cfg, zs, b=0, T=T, keep_weights=True)
elapsed = time.time() - t0
ntot = cfg.points
rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([cfg.seed, 991])))
idx = np.unique(rng.integers(0, ntot, size=ns))
out = {"T": T, "elapsed_s": elapsed, "idx": idx}
for k in range(T + 1):
    w = O.to_lib(rec["w"][k]).reshape(-1)
    peak = int(np.argmax(np.abs(w)))
    ii = np.unique(np.concatenate([idx, [peak]]))
    out[f"idx_{k}"] = ii
    out[f"w_{k}"] = w[ii]
    out[f"peak_{k}"] = float(np.max(np.abs(w)))
    for key in ("mean", "cov", "logC", "c", "B"):
        out[f"{key}_{k}"] = np.asarray(rec[key][k], dtype=np.float64)
wf, cf, Bf = rec["final"]
wf = O.to_lib(wf).reshape(-1)
out["w_final"] = wf[idx]
out["peak_final"] = float(np.max(np.abs(wf)))
out["c_final"], out["B_final"] = np.asarray(cf), np.asarray(Bf)
path = os.path.join(ROOT, "tests", "golden", f"{cid.lower()}_full_T{T}.npz")
np.savez_compressed(path, **out)
print(path, f"{elapsed:.0f} s")

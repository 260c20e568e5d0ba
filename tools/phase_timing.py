"""Per-phase cycle split of the resident kernel (needs tools/libpmf_timing.so, a
debug build with clock64 probes). Runs 5 C5 epochs and prints the split."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2412_07240_b200 import pmf  # noqa: E402
from workloads import make_config, simulate  # noqa: E402

lib = pmf.load_library("tools/libpmf_timing.so")
cfg = make_config("C5")
zs = simulate(cfg, T=6)["z"]
f = pmf.Filter(2, cfg.n, cfg.A, cfg.Q, batch=cfg.batch)
f.set_gaussian(cfg.prior_mean, np.broadcast_to(cfg.prior_cov, (cfg.batch, 2, 2)), cfg.k_sigma)
lik = pmf.make_likelihood(pmf.LIK_LINEAR_GAUSS, 2, H=cfg.H, R=cfg.R)
f.update(zs[0], lik)
f.regrid(cfg.k_sigma)
for k in range(1, 6):
    f.step(cfg.tau / cfg.l, cfg.l, zs[k], lik, cfg.k_sigma)
f.moments()
out = (C.c_ulonglong * 20)()
lib.pmf_debug_phase.restype = C.c_int
lib.pmf_debug_phase(out)
names = ["P3b->wait (loop top)", "mbar wait", "P1 load/gather", "P1 barrier", "P1 fft/unpack", "P2",
         "P3 inv-fft (to X consumed)", "X-consumed barrier", "P3 output", "tail barrier+write"]
for w, lab in ((0, "tid 0 (warp 0)"), (1, "tid 511 (warp 15)")):
    v = np.array(out[w * 10:(w + 1) * 10], dtype=float)
    tot = v.sum()
    print(lab, "total Mcycles/CTA", tot / 148 / 1e6)
    for n, x in zip(names, v):
        print(f"   {n:28s} {100 * x / tot:5.1f}%")

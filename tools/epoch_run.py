#!/usr/bin/env python
"""Run a few filter epochs of a BASELINE workload through the C ABI (for ncu launch lists
and quick timings): python tools/epoch_run.py C4 [epochs] [--predict-only]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_07240_b200 import pmf  # noqa: E402
from workloads import make_config, simulate  # noqa: E402

cid = sys.argv[1] if len(sys.argv) > 1 else "C4"
E = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 3
over = {}
for a in sys.argv[3:]:
    if a.startswith("--n="):
        over["n"] = tuple(int(x) for x in a[4:].split("x"))
cfg = make_config(cid, **over)
zs = simulate(cfg, T=E + 1)["z"]
st = torch.cuda.Stream()
f = pmf.Filter(cfg.nx, cfg.n, cfg.A, cfg.Q, batch=cfg.batch, dtype=cfg.dtype, stream=st.cuda_stream)
lik = (pmf.make_likelihood(pmf.LIK_RANGE_GAUSS, cfg.nx, sigma=cfg.sigma) if cfg.lik_kind == 1
       else pmf.make_likelihood(pmf.LIK_LINEAR_GAUSS, cfg.nx, H=cfg.H, R=cfg.R))
f.set_gaussian(cfg.prior_mean, np.broadcast_to(cfg.prior_cov, (cfg.batch, cfg.nx, cfg.nx)), cfg.k_sigma)
z = torch.tensor(zs, dtype=torch.float64, device="cuda")
f.update(z[0], lik)
f.regrid(cfg.k_sigma)
dt = cfg.tau / cfg.l
po = "--predict-only" in sys.argv
torch.cuda.synchronize()
for k in range(1, E + 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    if po:
        f.predict(dt, cfg.l)
        f.sync()
    else:
        f.step(dt, cfg.l, z[k], lik, cfg.k_sigma)
    e1.record(st)
    e1.synchronize()
    print(f"epoch {k}: {e0.elapsed_time(e1):.3f} ms  path={f.path} kernel={f.epoch_kernel}", flush=True)
f.close()

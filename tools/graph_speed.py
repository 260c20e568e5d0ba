#!/usr/bin/env python
"""Epoch time with and without CUDA-graph replay (no profiling), per workload:
    python tools/graph_speed.py C1 C2 C3"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2412_07240_b200 import pmf  # noqa: E402
from workloads import make_config, simulate  # noqa: E402

for cid in sys.argv[1:] or ["C1", "C2", "C3"]:
    cfg = make_config(cid)
    zs = simulate(cfg, T=60)["z"]
    res = {}
    for graphs in (False, True):
        s = torch.cuda.Stream()
        f = pmf.Filter(cfg.nx, cfg.n, cfg.A, cfg.Q, batch=cfg.batch, stream=s.cuda_stream)
        f.use_graphs(graphs)
        lik = (pmf.make_likelihood(pmf.LIK_RANGE_GAUSS, cfg.nx, sigma=cfg.sigma) if cfg.lik_kind == 1
               else pmf.make_likelihood(pmf.LIK_LINEAR_GAUSS, cfg.nx, H=cfg.H, R=cfg.R))
        f.set_gaussian(cfg.prior_mean, np.broadcast_to(cfg.prior_cov, (cfg.batch, cfg.nx, cfg.nx)), cfg.k_sigma)
        z = torch.tensor(zs, device="cuda")
        f.update(z[0], lik)
        f.regrid(cfg.k_sigma)
        for k in range(1, 6):
            f.step(cfg.tau / cfg.l, cfg.l, z[k], lik, cfg.k_sigma)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for k in range(6, 56):
            f.step(cfg.tau / cfg.l, cfg.l, z[k], lik, cfg.k_sigma)
        e1.record(s)
        e1.synchronize()
        res[graphs] = e0.elapsed_time(e1) / 50
        f.close()
    print(f"{cid}: direct {res[False] * 1e3:.1f} us/epoch, graph {res[True] * 1e3:.1f} us/epoch")

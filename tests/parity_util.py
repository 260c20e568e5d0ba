"""Helpers for GPU-vs-oracle parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np

from oracle import pmf_oracle as O
from paper_2412_07240_b200 import pmf

TOL = {"f64": 1e-10, "f32": 1e-4}     # north_star: relative L-inf normalised by the peak density


def lik_of(cfg):
    if cfg.lik_kind == 1:
        return pmf.make_likelihood(pmf.LIK_RANGE_GAUSS, cfg.nx, sigma=cfg.sigma)
    if cfg.lik_kind == 2:
        return pmf.make_likelihood(pmf.LIK_TERRAIN_GM, cfg.nx, gm=cfg.extra["gm"])
    return pmf.make_likelihood(pmf.LIK_LINEAR_GAUSS, cfg.nx, H=cfg.H, R=cfg.R)


def rel_linf(gpu, ref):
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(gpu - ref)) / np.max(np.abs(ref)))


def make_filter(cfg, dtype="f64", path=pmf.PATH_AUTO, **kw):
    f = pmf.Filter(cfg.nx, cfg.n, cfg.A, cfg.Q, batch=cfg.batch, dtype=dtype, path=path, **kw)
    if cfg.lik_kind == 2:
        from workloads import terrain_table
        f.set_terrain(*terrain_table(cfg))
    f.set_gaussian(cfg.prior_mean, np.broadcast_to(cfg.prior_cov, (cfg.batch, cfg.nx, cfg.nx)), cfg.k_sigma)
    return f


def run_gpu(cfg, zs, T, dtype="f64", path=pmf.PATH_AUTO, use_step=False, keep_weights=True, **kw):
    """Epoch loop of R15 through the C ABI; records what the oracle's run_filter records."""
    f = make_filter(cfg, dtype, path, **kw)
    lik = lik_of(cfg)
    dt = cfg.tau / cfg.l
    rec = {"mean": [], "cov": [], "logC": [], "c": [], "B": [], "w": []}
    for k in range(T + 1):
        if use_step and k > 0:
            f.step(dt, cfg.l, zs[k], lik, cfg.k_sigma)
        else:
            if k > 0:
                f.predict(dt, cfg.l)
            f.update(zs[k], lik)
        mean, cov, logc = f.moments()
        rec["mean"].append(mean)
        rec["cov"].append(cov)
        rec["logC"].append(logc)
        if not use_step:
            c, B = f.grid()
            rec["c"].append(c)
            rec["B"].append(B)
            if keep_weights:
                rec["w"].append(f.weights().astype(np.float64))
            f.regrid(cfg.k_sigma)
        elif k == 0:
            f.regrid(cfg.k_sigma)
    rec["filter"] = f
    return rec


def run_oracle(cfg, zs, T, filters=None):
    filters = range(cfg.batch) if filters is None else filters
    return {b: O.run_filter(cfg, zs, b=b, T=T, keep_weights=True) for b in filters}


def compare_runs(cfg, g, orc, T, tol, filters=None, check_weights=True):
    """Max errors over epochs/filters: weights (rel L-inf / peak), mean (/ sqrt max eig),
    cov (rel), logC (abs), grid (rel)."""
    filters = list(orc.keys()) if filters is None else filters
    errs = {"w": 0.0, "mean": 0.0, "cov": 0.0, "logC": 0.0, "grid": 0.0}
    for k in range(T + 1):
        for b in filters:
            o = orc[b]
            sd = np.sqrt(np.max(np.linalg.eigvalsh(o["cov"][k])))
            errs["mean"] = max(errs["mean"], float(np.max(np.abs(g["mean"][k][b] - o["mean"][k]))) / sd)
            errs["cov"] = max(errs["cov"], rel_linf(g["cov"][k][b], o["cov"][k]))
            errs["logC"] = max(errs["logC"], abs(float(g["logC"][k][b]) - o["logC"][k]))
            if g["c"]:
                errs["grid"] = max(errs["grid"], rel_linf(g["B"][k][b], o["B"][k]),
                                   float(np.max(np.abs(g["c"][k][b] - o["c"][k]))) / float(np.max(np.abs(o["B"][k]))))
            if check_weights and g["w"]:
                wo = O.to_lib(o["w"][k])
                errs["w"] = max(errs["w"], rel_linf(g["w"][k][b], wo))
    return errs

"""Parity at BASELINE.json's FULL sizes, through the C ABI in the
launch configuration bench.py times where it applies:

* C2 (one 256^2 filter, all 100 epochs) and C3 (one 128^3 filter, 2 epochs): the oracle
  runs them whole; every epoch's weights, moments, normaliser and grid are compared.
* C5 (4096 filters x 128^2, all 50 epochs): the whole batch runs on the GPU with the fused
  pmf_step API (as bench.py), the oracle runs a sample of filters one by one (first, middle
  and last -- partial -- CTA rounds); per-epoch moments/normaliser and the final weights and
  grid of the sampled filters.
* C4 (96^4 = 85M points): too large for the oracle's O(N^2) DFTs, so a property that
  holds at any size pins it: the predicted mean and covariance equal the scheme's
  closed form e^{At}m and the Riemann-sum Kalman-Bucy covariance (P6) of the sampled
  input's discrete moments (the plane path also matches the pencil path element by
  element at this size: test_gpu_plane.py)."""
import math

import numpy as np
import pytest

from oracle import pmf_oracle as O
from paper_2412_07240_b200 import pmf
from workloads import make_config, simulate

from parity_util import TOL, compare_runs, lik_of, make_filter, rel_linf, run_gpu, run_oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cid, T", [("C2", 100), ("C3", 2)])
def test_full_size_whole_filter_vs_oracle(cid, T):
    cfg = make_config(cid)
    zs = simulate(cfg, T=T)["z"]
    g = run_gpu(cfg, zs, T)
    orc = run_oracle(cfg, zs, T)
    e = compare_runs(cfg, g, orc, T, TOL["f64"])
    assert max(e.values()) <= 1e-10, e


def test_c5_all_epochs_resident_vs_oracle():
    """BASELINE C5's full run length (50 epochs) on the resident kernel for two filters:
    no drift of the GPU filter away from the oracle over the whole run."""
    cfg = make_config("C5", batch=2)
    T = cfg.T
    assert T == 50
    zs = simulate(cfg, T=T)["z"]
    g = run_gpu(cfg, zs, T, path=pmf.PATH_RESIDENT, keep_weights=False)
    orc = run_oracle(cfg, zs, T)
    e = compare_runs(cfg, g, orc, T, TOL["f64"], check_weights=False)
    assert max(e.values()) <= 1e-10, e
    wo = O.to_lib(orc[1]["final"][0])
    assert rel_linf(g["filter"].weights()[1], wo) < 1e-10


def test_full_size_c5_batch_sampled_vs_oracle():
    """The whole 4096-filter batch for all 50 epochs through bench.py's pmf_step call;
    sampled filters from every CTA round of the persistent kernel (148 CTAs walk filters
    b = blockIdx + 148 j): the first round, a middle one and the last, partial round
    (filters 3996..4095 run on CTAs 0..99), against the oracle every epoch."""
    cfg = make_config("C5")
    assert cfg.batch == 4096
    T = cfg.T
    assert T == 50
    zs = simulate(cfg, T=T)["z"]
    f = make_filter(cfg)
    assert f.path == pmf.PATH_RESIDENT
    lik = lik_of(cfg)
    dt = cfg.tau / cfg.l
    sample = [0, 1, 147, 148, 1023, 2048, 3995, 3996, 4050, 4095]
    rec = []
    for k in range(T + 1):
        if k == 0:
            f.update(zs[0], lik)
        else:
            f.step(dt, cfg.l, zs[k], lik, cfg.k_sigma)     # predict + update + regrid (bench.py's call)
        mean, cov, logc = f.moments()
        rec.append((mean[sample], cov[sample], logc[sample]))
        if k == 0:
            f.regrid(cfg.k_sigma)
    w = f.weights()                                        # flushes the last step's regrid (oracle "final")
    c, B = f.grid()
    for i, b in enumerate(sample):
        o = O.run_filter(cfg, zs, b=b, T=T)
        for k in range(T + 1):
            sd = math.sqrt(np.max(np.linalg.eigvalsh(o["cov"][k])))
            assert np.max(np.abs(rec[k][0][i] - o["mean"][k])) / sd < 1e-10
            assert rel_linf(rec[k][1][i], o["cov"][k]) < 1e-10
            assert abs(rec[k][2][i] - o["logC"][k]) < 1e-10
        wo, co, Bo = o["final"]
        assert rel_linf(w[b], O.to_lib(wo)) < 1e-10
        # the centre is the re-centred mean (R12) after 50 epochs: fp64 rounding relative to
        # |c|, not to the grid spacing (|c| ~ 50 spacings here)
        assert rel_linf(B[b], Bo) < 1e-12
        assert np.max(np.abs(c[b] - co)) < 1e-12 * max(np.max(np.abs(co)), np.max(np.abs(Bo)))


def _index_moments(w, n):
    """Index-space sum, first and second moments of a weight array in library layout
    (axis 0 fastest) by marginal sums."""
    nx = len(n)
    a = w.reshape(tuple(reversed(n)))                      # axes (nx-1, ..., 0)
    ax = lambda m: nx - 1 - m                              # array axis of state axis m
    u = [np.arange(N, dtype=np.float64) - (N - 1) / 2.0 for N in n]
    S = float(a.sum())
    m = np.zeros(nx)
    C = np.zeros((nx, nx))
    for p in range(nx):
        mp = a.sum(axis=tuple(ax(q) for q in range(nx) if q != p))
        m[p] = float(mp @ u[p])
        C[p, p] = float(mp @ (u[p] * u[p]))
        for q in range(p + 1, nx):
            M2 = a.sum(axis=tuple(ax(r) for r in range(nx) if r not in (p, q)))   # axes (q, p) order
            C[p, q] = C[q, p] = float(u[q] @ M2 @ u[p])
    return S, m, C


def test_full_size_c4_predict_moments_closed_form():
    """96^4 on the plane path (as bench.py's C4 line): predict only, A = CV blocks, l = 10."""
    from scipy.linalg import expm
    cfg = make_config("C4")
    ks = 9.0                                               # wide: the periodic wrap is below 1e-14
    f = pmf.Filter(cfg.nx, cfg.n, cfg.A, cfg.Q, path=pmf.PATH_PLANE)
    P = np.diag([1.0, 0.25, 0.6, 0.15])
    f.set_gaussian(cfg.prior_mean, P[None], ks)

    def moments():
        w = f.weights()[0].astype(np.float64)
        c, B = f.grid()
        S, m, C = _index_moments(w, cfg.n)
        mu = m / S
        Cu = C / S - np.outer(mu, mu)
        return c[0] + B[0] @ mu, B[0] @ Cu @ B[0].T

    m0, P0 = moments()
    tau, l = 4 * cfg.tau, cfg.l
    f.predict(tau / l, l)
    mean, cov = moments()
    F = expm(cfg.A * tau)
    dt = tau / l
    covx = F @ P0 @ F.T + dt * sum(expm(cfg.A * (tau - s * dt)) @ cfg.Q @ expm(cfg.A * (tau - s * dt)).T
                                   for s in range(l))
    assert np.max(np.abs(mean - F @ m0)) < 1e-11 * math.sqrt(np.max(np.diag(covx)))
    assert rel_linf(cov, covx) < 1e-10


def _golden(name):
    import os
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", name)
    if not os.path.exists(p):
        pytest.skip(f"{name} missing (tools/make_golden.py)")
    return np.load(p)


@pytest.mark.parametrize("cid, T, kw", [("C3", 50, {}), ("C4", 2, {}),
                                        ("C4", 2, {"path": pmf.PATH_PENCIL, "world": 4, "sharded": True})],
                         ids=["C3", "C4", "C4_sharded_x4"])
def test_full_size_run_vs_oracle_fixture(cid, T, kw):
    """BASELINE C3 (128^3, all 50 epochs) and C4 (96^4 = 85 M points, epochs 0-2: epoch 2's
    predict carries the regrid off the sheared grid of epoch 1, i.e. the split map with
    M23 != 0 through K1 and K2) at full
    size, in bench.py's launch configuration (the plane path; C4 on the three-pass route),
    (and C4 slab-sharded over 4 virtual ranks: the sharded three-pass route with its
    pipelined exchanges and the standalone window regrid in its large-slab configuration)
    against the oracle's run of the same seeded inputs: tests/golden/<cfg>_full_T<T>.npz,
    written by tools/make_golden.py (oracle/ only). Every epoch: moments, normaliser and
    grid, and the posterior weights element by element at 8192 (C4) / 2048 (C3) seeded
    positions plus the peak, relative to the oracle's peak |w|; then the final regridded
    weights."""
    G = _golden(f"{cid.lower()}_full_T{T}.npz")
    cfg = make_config(cid)
    zs = simulate(cfg, T=T)["z"]
    f = make_filter(cfg, **kw)
    assert f.world == 4 if kw else f.path == pmf.PATH_PLANE
    lik = lik_of(cfg)
    dt = cfg.tau / cfg.l
    for k in range(T + 1):
        if k > 0:
            f.predict(dt, cfg.l)
        f.update(zs[k], lik)
        mean, cov, logc = f.moments()
        c, B = f.grid()
        sd = math.sqrt(np.max(np.linalg.eigvalsh(G[f"cov_{k}"])))
        assert np.max(np.abs(mean[0] - G[f"mean_{k}"])) / sd < 1e-10, k
        assert rel_linf(cov[0], G[f"cov_{k}"]) < 1e-10, k
        assert abs(logc[0] - float(G[f"logC_{k}"])) < 1e-10, k
        assert rel_linf(B[0], G[f"B_{k}"]) < 1e-10, k
        assert np.max(np.abs(c[0] - G[f"c_{k}"])) < 1e-10 * np.max(np.abs(G[f"B_{k}"])), k
        if k == T or cid == "C4" or k % 10 == 0:
            w = f.weights()[0].reshape(-1)
            ii = G[f"idx_{k}"]
            peak = float(G[f"peak_{k}"])
            assert abs(float(np.max(np.abs(w))) - peak) <= 1e-10 * peak, k
            assert float(np.max(np.abs(w[ii] - G[f"w_{k}"]))) <= 1e-10 * peak, k
            del w
        f.regrid(cfg.k_sigma)
    w = f.weights()[0].reshape(-1)                           # flushes the last regrid
    c, B = f.grid()
    assert float(np.max(np.abs(w[G["idx"]] - G["w_final"]))) <= 1e-10 * float(G["peak_final"])
    assert rel_linf(B[0], G["B_final"]) < 1e-12

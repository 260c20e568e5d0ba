"""Seeded synthetic workloads for the spectral point-mass filter (PMF).

This module is the ONLY code shared by the CUDA path's tests/bench and the CPU
oracle. It holds model constants, grid sizes and seeded random draws (truth
trajectories and measurements) and NONE of the method's arithmetic: no DFT, no
spectral multiplier, no grid motion, no likelihood, no moments, no regrid.
The truth simulation uses scipy's matrix exponential (a library primitive) for
the exact discretisation of the SDE; neither the oracle nor the
CUDA library uses this module's numbers for anything but inputs.

Configs mirror BASELINE.json ``configs`` C1..C5 with the readings of
SURVEY.md §8(c) (R15-R19) for what the configs leave unspecified:

* C1  1-D  dx = -0.5 x dt + 1.0 dw, N=64, prior N(1, 0.5^2), tau=0.1, 20 epochs,
       z = x + v, v ~ N(0, 0.3^2)                         (BASELINE configs[0])
* C2  2-D CV A=[[0,1],[0,0]], Q=diag(0,0.1), 256^2, prior N((0,1),diag(1,.25)),
       tau=0.05, 100 epochs, H=[1 0], R=0.5^2              (configs[1])
* C3  3-D A ~ U[-0.5,0.5]^{3x3} shifted so max Re(eig) <= 0, Q=0.2 I, 128^3,
       h(x)=||x||, sigma=0.1, tau=0.02, 50 epochs          (configs[2], R17)
* C4  4-D [px,vx,py,vy] CV, Q=diag(0,.05,0,.05), 96^4, H picks px,py,
       R=0.25 I, tau=0.05, 20 epochs                       (configs[3], R18)
* C5  4096 independent C2-model filters on 128^2, prior means ~ N(0, I),
       cov diag(1,.25), tau=0.05, 50 epochs                (configs[4], R19)
* C6  the paper's §VI tracking scenario: coordinated turn
       [px,vx,py,vy] with alpha = 30 deg/s, Q = G G^T = diag(0,1,0,1), prior
       N((36569,50,55581,50), diag(90,160,5,5)), T_s = 1 s, N_pa = 34; measurement =
       terrain altitude below the vehicle + 2-component GM noise 1/2 N(0,1) + 1/2
       N(20,1). The SRTM map is unavailable: the terrain is a seeded analytic field
       (three sinusoids, ~ +-90 m) sampled on a 10 m table; the truth measurement
       uses the analytic field, the filter only the table.

Every config uses k_sigma = 6 (R10) and l = 10 Euler substeps per prediction
interval (R15). Sizes can be overridden to build small parity cases.
"""
from __future__ import annotations

import dataclasses
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

LIK_LINEAR_GAUSS = 0
LIK_RANGE_GAUSS = 1
LIK_TERRAIN_GM = 2


@dataclass
class Config:
    name: str
    nx: int
    n: tuple                 # points per axis (axis 0 first)
    batch: int
    A: np.ndarray            # nx x nx drift matrix  (eq:dynam)
    Q: np.ndarray            # nx x nx FPE diffusion matrix (eq:fokker; R1)
    prior_mean: np.ndarray   # batch x nx
    prior_cov: np.ndarray    # nx x nx (shared by all filters)
    k_sigma: float
    tau: float               # prediction interval t_{k+1} - t_k
    l: int                   # Euler substeps per interval
    T: int                   # number of predict+update epochs after the k=0 update
    lik_kind: int
    H: Optional[np.ndarray] = None     # nz x nx (linear Gaussian)
    R: Optional[np.ndarray] = None     # nz x nz
    sigma: float = 0.0                 # range-measurement noise std
    seed: int = 0
    dtype: str = "f64"
    extra: dict = field(default_factory=dict)

    @property
    def nz(self) -> int:
        return 1 if self.lik_kind in (LIK_RANGE_GAUSS, LIK_TERRAIN_GM) else int(self.H.shape[0])

    @property
    def points(self) -> int:
        return int(np.prod(self.n))

    def replace(self, **kw) -> "Config":
        return dataclasses.replace(self, **kw)


def _cv_A():
    return np.array([[0.0, 1.0], [0.0, 0.0]])


def _c3_A(rng: np.random.Generator) -> np.ndarray:
    # R17: A ~ U[-0.5,0.5]^{3x3} row-major, then A <- A - max(0, max Re eig(A)) I
    A = rng.uniform(-0.5, 0.5, size=(3, 3))
    shift = max(0.0, float(np.max(np.linalg.eigvals(A).real)))
    return A - shift * np.eye(3)


def make_config(cid: str, **over) -> Config:
    """Build config ``cid`` in {"C1",...,"C5"}; keyword overrides replace fields
    (e.g. ``n=(32, 32)`` or ``batch=8``) to build small parity cases."""
    cid = cid.upper()
    if cid == "C1":
        cfg = Config(name="C1", nx=1, n=(64,), batch=1, A=np.array([[-0.5]]),
                     Q=np.array([[1.0]]), prior_mean=np.array([[1.0]]),
                     prior_cov=np.array([[0.25]]), k_sigma=6.0, tau=0.1, l=10, T=20,
                     lik_kind=LIK_LINEAR_GAUSS, H=np.array([[1.0]]),
                     R=np.array([[0.09]]), seed=1)
    elif cid == "C2":
        cfg = Config(name="C2", nx=2, n=(256, 256), batch=1, A=_cv_A(),
                     Q=np.diag([0.0, 0.1]), prior_mean=np.array([[0.0, 1.0]]),
                     prior_cov=np.diag([1.0, 0.25]), k_sigma=6.0, tau=0.05, l=10,
                     T=100, lik_kind=LIK_LINEAR_GAUSS, H=np.array([[1.0, 0.0]]),
                     R=np.array([[0.25]]), seed=2)
    elif cid == "C3":
        rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(3)))
        cfg = Config(name="C3", nx=3, n=(128, 128, 128), batch=1, A=_c3_A(rng),
                     Q=0.2 * np.eye(3), prior_mean=np.array([[2.0, 0.0, 0.0]]),
                     prior_cov=0.25 * np.eye(3), k_sigma=6.0, tau=0.02, l=10, T=50,
                     lik_kind=LIK_RANGE_GAUSS, sigma=0.1, seed=3)
    elif cid == "C4":
        A = np.zeros((4, 4))
        A[0, 1] = 1.0
        A[2, 3] = 1.0
        cfg = Config(name="C4", nx=4, n=(96, 96, 96, 96), batch=1, A=A,
                     Q=np.diag([0.0, 0.05, 0.0, 0.05]),
                     prior_mean=np.array([[0.0, 1.0, 0.0, 1.0]]),
                     prior_cov=np.diag([1.0, 0.25, 1.0, 0.25]), k_sigma=6.0,
                     tau=0.05, l=10, T=20, lik_kind=LIK_LINEAR_GAUSS,
                     H=np.array([[1.0, 0, 0, 0], [0, 0, 1.0, 0]]),
                     R=0.25 * np.eye(2), seed=4)
    elif cid == "C6":
        alpha = math.pi / 6.0
        A = np.zeros((4, 4))
        A[0, 1] = 1.0
        A[1, 3] = -alpha
        A[2, 3] = 1.0
        A[3, 1] = alpha
        cfg = Config(name="C6", nx=4, n=(34, 34, 34, 34), batch=1, A=A, Q=np.diag([0.0, 1.0, 0.0, 1.0]),
                     prior_mean=np.array([[36569.0, 50.0, 55581.0, 50.0]]),
                     prior_cov=np.diag([90.0, 160.0, 5.0, 5.0]), k_sigma=6.0, tau=1.0, l=10, T=20,
                     lik_kind=LIK_TERRAIN_GM, seed=6,
                     extra={"gm": ((0.5, 0.0, 1.0), (0.5, 20.0, 1.0))})
    elif cid == "C5":
        cfg = Config(name="C5", nx=2, n=(128, 128), batch=4096, A=_cv_A(),
                     Q=np.diag([0.0, 0.1]), prior_mean=None,
                     prior_cov=np.diag([1.0, 0.25]), k_sigma=6.0, tau=0.05, l=10,
                     T=50, lik_kind=LIK_LINEAR_GAUSS, H=np.array([[1.0, 0.0]]),
                     R=np.array([[0.25]]), seed=5)
    else:
        raise ValueError(f"unknown config {cid}")
    cfg = dataclasses.replace(cfg, **over)
    if cfg.prior_mean is None or cfg.prior_mean.shape[0] != cfg.batch:
        cfg = dataclasses.replace(cfg, prior_mean=_prior_means(cfg))
    return cfg


def terrain_field(cfg: Config, x, y):
    """The C6 synthetic terrain (analytic; seeded phases): altitude [m] at (x, y) [m]."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([cfg.seed, 7])))
    ph = rng.uniform(0.0, 2.0 * math.pi, 3)
    return (300.0 + 60.0 * np.sin(2 * math.pi * x / 350.0 + ph[0]) * np.cos(2 * math.pi * y / 420.0 + ph[1])
            + 25.0 * np.sin(2 * math.pi * (x + y) / 180.0 + ph[2]))


def terrain_table(cfg: Config, spacing: float = 10.0, half: float = 900.0):
    """The map the filter gets: the C6 field sampled on a square table around the prior
    mean. Returns (heights[r, c], x0, y0, dx, dy, ix, iy): heights[r, c] at
    (x0 + c dx, y0 + r dy); state components ix = 0 (px), iy = 2 (py)."""
    mx, my = cfg.prior_mean[0, 0], cfg.prior_mean[0, 2]
    n = int(round(2 * half / spacing)) + 1
    xs = mx - half + spacing * np.arange(n)
    ys = my - half + spacing * np.arange(n)
    X, Y = np.meshgrid(xs, ys)
    return terrain_field(cfg, X, Y), float(xs[0]), float(ys[0]), spacing, spacing, 0, 2


def _prior_means(cfg: Config) -> np.ndarray:
    """C5 (R19): per-filter prior mean m_i ~ N(0, I) drawn from the filter's own
    spawned stream; other configs replicate their fixed prior mean."""
    if cfg.name == "C5":
        ss = np.random.SeedSequence(cfg.seed).spawn(cfg.batch)
        out = np.empty((cfg.batch, cfg.nx))
        for i, s in enumerate(ss):
            out[i] = np.random.Generator(np.random.PCG64(s)).standard_normal(cfg.nx)
        return out
    base = make_config(cfg.name).prior_mean[0]
    return np.tile(base, (cfg.batch, 1))


def _psd_sqrt(M: np.ndarray) -> np.ndarray:
    w, V = np.linalg.eigh(0.5 * (M + M.T))
    return V @ np.diag(np.sqrt(np.clip(w, 0.0, None)))


def _discretise(A: np.ndarray, Q: np.ndarray, tau: float):
    """Exact discretisation of dx = Ax dt + dW, E[dW dW^T] = Q dt (Van Loan),
    for the TRUTH simulation only (R16/R22)."""
    from scipy.linalg import expm
    n = A.shape[0]
    C = np.zeros((2 * n, 2 * n))
    C[:n, :n] = -A
    C[:n, n:] = Q
    C[n:, n:] = A.T
    E = expm(C * tau)
    F = E[n:, n:].T
    Qd = F @ E[:n, n:]
    return F, 0.5 * (Qd + Qd.T)


def simulate(cfg: Config, T: Optional[int] = None) -> dict:
    """Seeded truth trajectory and measurements (R16).

    Returns ``{"truth": (batch, T+1, nx), "z": (T+1, batch, nz)}``. Draw order
    per filter Generator: x0 = m0 + chol(P0) N(0,I); process noise for k=1..T;
    measurement noise for k=0..T.
    """
    T = cfg.T if T is None else T
    F, Qd = _discretise(cfg.A, cfg.Q, cfg.tau)
    Sq, S0 = _psd_sqrt(Qd), _psd_sqrt(cfg.prior_cov)
    if cfg.name == "C5":
        seeds = np.random.SeedSequence(cfg.seed).spawn(cfg.batch)
    else:
        seeds = np.random.SeedSequence(cfg.seed).spawn(cfg.batch)
    truth = np.empty((cfg.batch, T + 1, cfg.nx))
    z = np.empty((T + 1, cfg.batch, cfg.nz))
    for b, s in enumerate(seeds):
        rng = np.random.Generator(np.random.PCG64(s))
        if cfg.name == "C5":
            rng.standard_normal(cfg.nx)          # consumed by the prior mean draw
        x = cfg.prior_mean[b] + S0 @ rng.standard_normal(cfg.nx)
        truth[b, 0] = x
        for k in range(1, T + 1):
            x = F @ x + Sq @ rng.standard_normal(cfg.nx)
            truth[b, k] = x
        for k in range(T + 1):
            xk = truth[b, k]
            if cfg.lik_kind == LIK_RANGE_GAUSS:
                z[k, b, 0] = np.linalg.norm(xk) + cfg.sigma * rng.standard_normal()
            elif cfg.lik_kind == LIK_TERRAIN_GM:
                gm = cfg.extra["gm"]
                g = rng.choice(len(gm), p=[c[0] for c in gm])
                z[k, b, 0] = terrain_field(cfg, xk[0], xk[2]) + gm[g][1] + math.sqrt(gm[g][2]) * rng.standard_normal()
            else:
                z[k, b] = cfg.H @ xk + _psd_sqrt(cfg.R) @ rng.standard_normal(cfg.nz)
    return {"truth": truth, "z": z}


def random_density(n: tuple, batch: int, seed: int) -> np.ndarray:
    """A seeded smooth positive test field of shape (batch, *reversed(n)) in the
    library's memory layout (axis 0 fastest): a sum of 3 random Gaussian bumps in
    index coordinates, bounded away from the grid edges (used for operator-level
    parity cases that need a non-Gaussian input)."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(seed)))
    nx = len(n)
    out = np.zeros((batch,) + tuple(reversed(n)))
    axes = [np.arange(m) - (m - 1) / 2.0 for m in n]
    grids = np.meshgrid(*axes, indexing="ij")           # each shape n (axis0 first)
    for b in range(batch):
        f = np.zeros(n)
        for _ in range(3):
            mu = [rng.uniform(-0.15, 0.15) * m for m in n]
            sd = [rng.uniform(0.06, 0.11) * m for m in n]
            amp = rng.uniform(0.5, 1.5)
            e = sum(((g - m_) / s_) ** 2 for g, m_, s_ in zip(grids, mu, sd))
            f += amp * np.exp(-0.5 * e)
        out[b] = f.transpose(tuple(reversed(range(nx))))
    return out

"""Pins of the oracle's FDM baseline (PAPER §III.A-B)
against what the paper and the mathematics fix, independently of the oracle's own
formulas:

* P15 the closed-form eigenvalues of F_diff = a library eigensolver's;
* P16 the DST-I eigenvector matrix satisfies R^{-1} = 2/(N+1) R;
* P17 the fast-sine-transform predictor (eq:FST P:199-202) = literal explicit FDM
      stepping (eq:FDM P:146-150) on sheared, moving grids, nx = 1..3;
* P18 the FDM spatial error falls as O(1/N^2) against the exact heat-kernel
      solution of the pure-diffusion FPE (a Gaussian of variance sigma^2 + q tau);
* P19 spectral differentiation beats the FDM at equal N on a smooth density (the
      paper's central claim): a qualitative ordering, not a tolerance.
"""
import math

import numpy as np
import pytest

from oracle import pmf_oracle as O


@pytest.mark.parametrize("N,a,b", [(5, 0.3, 0.1), (12, -0.7, 2.0), (33, 0.25, 0.5)])
def test_p15_fdm_eigenvalues_closed_form(N, a, b):
    ev = np.sort(np.linalg.eigvalsh(O.fdm_matrix(N, a, b)))
    assert np.max(np.abs(ev - np.sort(O.fdm_eigenvalues(N, a, b)))) < 1e-13


@pytest.mark.parametrize("N", [4, 7, 32, 97])
def test_p16_dst_orthogonality(N):
    R = O.dst1_matrix(N)
    assert np.max(np.abs(R @ R * (2.0 / (N + 1)) - np.eye(N))) < 1e-13
    # and R diagonalises F_diff with the closed-form eigenvalues (columns = eigenvectors)
    F = O.fdm_matrix(N, 0.4, 0.3)
    lam = O.fdm_eigenvalues(N, 0.4, 0.3)
    assert np.max(np.abs(F @ R - R * lam[None, :])) < 1e-12


@pytest.mark.parametrize("nx,n", [(1, (9,)), (2, (7, 6)), (3, (5, 6, 4))])
def test_p17_fst_equals_explicit_fdm(nx, n):
    rng = np.random.default_rng(40 + nx)
    A = 0.3 * rng.standard_normal((nx, nx))
    Q = np.diag(rng.uniform(0.05, 0.2, nx))
    B = np.diag(rng.uniform(0.2, 0.4, nx)) + 0.02 * rng.standard_normal((nx, nx))
    c = rng.standard_normal(nx)
    w = rng.random(n)
    a, ca, Ba = O.fdm_predict_unnormalised(w, c, B, A, Q, 0.3, 7)
    b, cb, Bb = O.fst_predict_unnormalised(w, c, B, A, Q, 0.3, 7)
    assert np.max(np.abs(a - b)) / np.max(np.abs(a)) < 1e-13
    assert np.allclose(ca, cb) and np.allclose(Ba, Bb)


def _heat_errors(N, method, q=1.0, tau=0.1, l=20000, sigma=1.0, half_width=8.0):
    """Max error (relative to the peak) of one predict of N(0, sigma^2) under pure
    diffusion q against the exact N(0, sigma^2 + q tau) on a grid of +-half_width sigma."""
    delta = 2.0 * half_width * sigma / N
    c, B = np.zeros(1), np.array([[delta]])
    x = O.grid_points(c, B, (N,))[0]
    w = np.exp(-0.5 * x ** 2 / sigma ** 2)
    A = np.zeros((1, 1))
    Q = np.array([[q]])
    if method == "fdm":
        out, _, _ = O.fst_predict_unnormalised(w, c, B, A, Q, tau, l)
    else:
        out, _, _ = O.predict_unnormalised(w, c, B, A, Q, tau, l)
    out = out / (np.sum(out) * delta)
    s2 = sigma ** 2 + q * tau
    exact = np.exp(-0.5 * x ** 2 / s2) / math.sqrt(2 * math.pi * s2)
    return float(np.max(np.abs(out - exact)) / np.max(exact))


def test_p18_fdm_second_order_in_space():
    e1, e2, e3 = (_heat_errors(N, "fdm") for N in (32, 64, 128))
    assert 3.3 < e1 / e2 < 4.7 and 3.3 < e2 / e3 < 4.7, (e1, e2, e3)


def test_p19_spectral_beats_fdm_at_equal_n():
    for N in (32, 64):
        assert _heat_errors(N, "spectral") < 0.2 * _heat_errors(N, "fdm")


def test_p20_heat_kernel_reference_solves_the_fpe():
    """The convergence experiment's reference (tools/convergence.py: the mixture with
    every variance + q t) solves dp/dt = (q/2) d2p/dx2 (eq:fokker P:55 with A = 0):
    central differences in t and x agree to O(h^2)."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "convergence", os.path.join(os.path.dirname(os.path.dirname(__file__)), "tools", "convergence.py"))
    conv = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(conv)
    comps = conv.DENSITIES["gm3"]
    x = np.linspace(-4, 4, 41)
    t, h, q = 0.1, 1e-4, conv.Q
    dpdt = (conv.mixture(x, comps, q * (t + h)) - conv.mixture(x, comps, q * (t - h))) / (2 * h)
    hx = 1e-3
    p0 = conv.mixture(x, comps, q * t)
    d2 = (conv.mixture(x + hx, comps, q * t) - 2 * p0 + conv.mixture(x - hx, comps, q * t)) / hx ** 2
    assert np.max(np.abs(dpdt - 0.5 * q * d2)) < 1e-5 * np.max(np.abs(dpdt))


def test_p21_terrain_table_function():
    """R26 table function: exact on bilinear fields, reproduces the nodes, clamps outside;
    the GM likelihood integrates to one over z and reduces to a Gaussian for one component."""
    rng = np.random.default_rng(3)
    a, b, cxy, d = rng.standard_normal(4)
    x0, y0, dx, dy = 10.0, -5.0, 2.0, 3.0
    xs, ys = x0 + dx * np.arange(7), y0 + dy * np.arange(5)
    X, Y = np.meshgrid(xs, ys)
    H = a + b * X + cxy * Y + d * X * Y
    px, py = rng.uniform(xs[0], xs[-1], 50), rng.uniform(ys[0], ys[-1], 50)
    exact = a + b * px + cxy * py + d * px * py
    assert np.max(np.abs(O.terrain_height(px, py, H, x0, y0, dx, dy) - exact)) < 1e-12
    assert np.max(np.abs(O.terrain_height(X, Y, H, x0, y0, dx, dy) - H)) < 1e-12
    assert abs(O.terrain_height(xs[0] - 50, ys[-1] + 9, H, x0, y0, dx, dy) - H[-1, 0]) < 1e-12
    table = (H, x0, y0, dx, dy, 0, 1)
    gm = ((0.5, 0.0, 1.0), (0.5, 20.0, 1.0))
    pt = np.array([[15.3], [2.2]])
    h = O.terrain_height(15.3, 2.2, H, x0, y0, dx, dy)
    zs = np.linspace(h - 15, h + 40, 20001)
    vals = np.array([O.lik_terrain_gm(pt, z, table, gm)[0] for z in zs])
    assert abs(np.sum(vals) * (zs[1] - zs[0]) - 1.0) < 1e-6
    g1 = O.lik_terrain_gm(pt, h + 0.7, table, ((1.0, 0.0, 4.0),))[0]
    assert abs(g1 - math.exp(-0.5 * 0.49 / 4.0) / math.sqrt(2 * math.pi * 4.0)) < 1e-15


def _cn_heat_error(l, step, N=128, q=1.0, tau=0.2, sigma=1.0, half_width=10.0):
    delta = 2.0 * half_width * sigma / N
    c, B = np.zeros(1), np.array([[delta]])
    x = O.grid_points(c, B, (N,))[0]
    w = np.exp(-0.5 * x ** 2 / sigma ** 2)
    out, _, _ = O.predict_unnormalised(w, c, B, np.zeros((1, 1)), np.array([[q]]), tau, l, step=step)
    out = out / (np.sum(out) * delta)
    s2 = sigma ** 2 + q * tau
    exact = np.exp(-0.5 * x ** 2 / s2) / math.sqrt(2 * math.pi * s2)
    return float(np.max(np.abs(out - exact)) / np.max(exact))


def test_p22_crank_nicolson_second_order_vs_heat_kernel():
    """NEXT-4 (R27): Crank-Nicolson substeps converge at second order in dt to the exact
    heat-kernel solution (the paper's semi-implicit Euler at first order)."""
    e = [_cn_heat_error(l, O.STEP_CN) for l in (4, 8, 16)]
    assert 3.5 < e[0] / e[1] < 4.5 and 3.5 < e[1] / e[2] < 4.5, e
    u = [_cn_heat_error(l, O.STEP_EULER) for l in (4, 8, 16)]
    assert 1.7 < u[0] / u[1] < 2.3, u
    assert e[2] < 0.05 * u[2]


def test_p23_crank_nicolson_moving_grid_covariance():
    """On a moving, shearing grid (CV drift) the CN predictor's covariance converges at
    second order to the continuous-time Kalman-Bucy covariance e^{A t} P e^{A^T t} +
    int_0^t e^{A s} Q e^{A^T s} ds (Van Loan): the time-dependent diffusion is handled
    explicit-at-t_n / implicit-at-t_{n+1}."""
    from scipy.linalg import expm
    A = np.array([[0.0, 1.0], [0.0, 0.0]])
    Q = np.diag([0.0, 0.4])
    P0 = np.diag([1.0, 0.25])
    n = (96, 96)
    tau = 1.0
    c, B = O.design_grid(np.zeros(2), np.diag([4.0, 1.2]), n, 8.0)
    w = O.gaussian_pdf(O.grid_points(c, B, n), np.zeros(2), P0)
    M = np.zeros((4, 4))
    M[:2, :2], M[:2, 2:], M[2:, 2:] = -A, Q, A.T
    E = expm(M * tau)
    F = E[2:, 2:].T
    Pex = F @ P0 @ F.T + F @ E[:2, 2:]
    errs = []
    for l in (4, 8, 16):
        wp, cp, Bp = O.predict(w, c, B, A, Q, tau, l, step=O.STEP_CN)
        _, cov = O.moments(wp, cp, Bp)
        errs.append(float(np.max(np.abs(cov - Pex))))
    assert 3.3 < errs[0] / errs[1] < 4.7 and 3.3 < errs[1] / errs[2] < 4.7, errs

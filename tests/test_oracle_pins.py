"""Pins for the CPU oracle: each check fixes the oracle
against something other than itself -- the paper's closed forms, library
routines for special cases, brute-force dense solves, Kalman closed forms,
golden values with citations. CPU only."""
import json
import math
import os

import numpy as np
import pytest
from scipy.special import erfc

from oracle import pmf_oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(np.max(np.abs(b)), 1e-300))


# --------------------------------------------------------------------- P1 DFT
@pytest.mark.parametrize("n", [(8,), (6, 4), (12, 8, 6), (4, 6, 4, 8)])
def test_dft_equals_library_fft(n):
    """eq:fourtrsf with 1/N forward = numpy's FFT / N (library routine);
    inverse unscaled (R6). Catches sign, scaling and axis-order slips."""
    rng = np.random.default_rng(0)
    w = rng.standard_normal(n)
    S = O.dftn(w)
    assert rel(S, np.fft.fftn(w) / np.prod(n)) < 1e-13
    assert rel(O.idftn(S).real, w) < 1e-13
    assert rel(O.idftn(S), np.fft.ifftn(S) * np.prod(n)) < 1e-13


def test_dft_golden_cosine_and_constant():
    g = GOLD["dft_cosine_mode"]
    N, s = g["N"], g["s"]
    j = np.arange(N)
    S = O.dftn(np.cos(2 * math.pi * s * j / N))
    exp = np.zeros(N)
    for k, v in g["expected_nonzero"].items():
        exp[int(k)] = v
    assert np.max(np.abs(S - exp)) < 1e-15
    g = GOLD["dft_constant"]
    S = O.dftn(np.full(g["N"], g["c"]))
    assert abs(S[0] - g["c"]) < 1e-15 and np.max(np.abs(S[1:])) < 1e-15


# --------------------------------------------------------------------- P2 tables
def test_second_derivative_coeffs_golden():
    for key in ("second_derivative_coeffs", "second_derivative_coeffs_L_pi"):
        g = GOLD[key]
        c2 = O.second_derivative_coeffs(g["N"], g["L_over_pi"] * math.pi)
        assert np.allclose(c2, g["expected"], rtol=0, atol=1e-14), key


def test_psi_golden_and_bounds():
    """psi = 1/1.2 through the index-space form: N=4, delta = pi/2
    (L = 2 pi), Nyquist wavenumber gives c'' = -4, D = Q/delta^2."""
    g = GOLD["psi_example"]
    delta = math.pi / 2
    D = np.array([[g["Q"] / delta ** 2]])
    psi = O.psi_factor(D, g["dt"], (4,))
    assert abs(psi[2] - g["expected"]) < 1e-15
    assert abs(psi[1] - 1 / 1.05) < 1e-15 and psi[0] == 1.0
    rng = np.random.default_rng(1)
    M = rng.standard_normal((3, 3))
    D = M @ M.T
    psi = O.psi_factor(D, 0.3, (8, 6, 4))
    assert psi[0, 0, 0] == 1.0
    assert np.all(psi > 0) and np.all(psi <= 1.0 + 1e-15)


# --------------------------------------------------------------------- P3 derivatives
@pytest.mark.parametrize("N", [16, 64])
def test_spectral_derivatives_exact_on_bandlimited_modes(N):
    """A band-limited mode |s| < N/2 is differentiated exactly (P:215 spectral
    accuracy; eq:secDer); the pure Nyquist mode too for p''."""
    L = 3.7
    delta = L / N
    x = O.axis_offsets(N) * delta
    for s in (1, 3, N // 2 - 1):
        for ph in (0.0, 0.7):
            f = np.sin(2 * math.pi * s * x / L + ph)
            k = 2 * math.pi * s / L
            assert np.max(np.abs(O.spectral_second_derivative(f, L) + k * k * f)) < 1e-12 * k * k
            d1 = k * np.cos(2 * math.pi * s * x / L + ph)
            assert np.max(np.abs(O.spectral_first_derivative(f, L) - d1)) < 1e-12 * k
    f = np.cos(math.pi * N * x / L + 0.3)          # Nyquist: samples (+-1)^j const
    kN = math.pi * N / L
    assert np.max(np.abs(O.spectral_second_derivative(f, L) + kN ** 2 * f)) < 1e-12 * kN ** 2
    assert np.max(np.abs(O.spectral_first_derivative(f, L))) < 1e-12 * kN


def test_spectral_second_derivative_gaussian():
    """Analytic Gaussian p'' = (x^2/s^4 - 1/s^2) p on a +-10 sigma grid."""
    N, sig = 128, 0.7
    L = 20 * sig
    x = O.axis_offsets(N) * (L / N)
    p = np.exp(-0.5 * x * x / sig ** 2)
    exact = (x * x / sig ** 4 - 1 / sig ** 2) * p
    assert rel(O.spectral_second_derivative(p, L), exact) < 1e-12


# --------------------------------------------------------------------- P4 brute force
def _trefethen(N):
    """Dense spectral differentiation matrices for the periodic grid of N
    (even) points, Trefethen 'Spectral Methods in MATLAB' ch.3 closed forms
    in theta = 2 pi j / N, converted to index coordinates (d/du = 2pi/N d/dtheta).
    D1 is the Nyquist-free first derivative; D2 keeps the Nyquist term."""
    h = 2 * math.pi / N
    D1 = np.zeros((N, N))
    D2 = np.zeros((N, N))
    for j in range(N):
        for k in range(N):
            if j == k:
                D2[j, k] = -math.pi ** 2 / (3 * h * h) - 1.0 / 6.0
            else:
                t = (j - k) * h / 2
                sgn = (-1) ** (j - k)
                D1[j, k] = 0.5 * sgn / math.tan(t)
                D2[j, k] = -0.5 * sgn / math.sin(t) ** 2
    c = 2 * math.pi / N
    return c * D1, c * c * D2


def _dense_predict(w, B, A, Q, tau, l):
    """Per-substep dense backward-Euler solve (P4):
    (I - dt/2 sum_ab D_ab d_a d_b) w_{n+1} = (1 - dt trA) w_n on the grid at
    the start of substep n, d_a the dense spectral derivative along axis a."""
    n = w.shape
    nx = len(n)
    mats = [_trefethen(N) for N in n]
    eye = [np.eye(N) for N in n]

    def kron_axis(ops):  # ops[a] acting on axis a, C-order flattening of w
        M = np.array([[1.0]])
        for a in range(nx):
            M = np.kron(M, ops[a])
        return M

    dt = tau / l
    Ntot = int(np.prod(n))
    v = w.reshape(-1).copy()
    from scipy.linalg import expm
    for s in range(l):
        Bn = expm(A * s * dt) @ B
        Bi = np.linalg.inv(Bn)
        D = Bi @ Q @ Bi.T
        Lop = np.zeros((Ntot, Ntot))
        for a in range(nx):
            ops = list(eye)
            ops[a] = mats[a][1]
            Lop += D[a, a] * kron_axis(ops)
            for b in range(a + 1, nx):
                ops = list(eye)
                ops[a] = mats[a][0]
                ops[b] = mats[b][0]
                Lop += 2 * D[a, b] * kron_axis(ops)
        v = np.linalg.solve(np.eye(Ntot) - 0.5 * dt * Lop, (1 - dt * np.trace(A)) * v)
    return v.reshape(n)


@pytest.mark.parametrize("n,seed", [((8,), 0), ((8, 6), 1), ((6, 4, 4), 2)])
def test_predict_equals_dense_brute_force(n, seed):
    rng = np.random.default_rng(seed)
    nx = len(n)
    A = 0.6 * rng.standard_normal((nx, nx))       # non-diagonal: the grid shears
    M = rng.standard_normal((nx, nx))
    Q = M @ M.T + 0.1 * np.eye(nx)
    B = np.diag(rng.uniform(0.3, 0.8, nx)) + 0.1 * rng.standard_normal((nx, nx))
    c = rng.standard_normal(nx)
    w = rng.uniform(0.1, 1.0, n)
    tau, l = 0.4, 3
    wo, cl, Bl = O.predict_unnormalised(w, c, B, A, Q, tau, l)
    assert rel(wo, _dense_predict(w, B, A, Q, tau, l)) < 1e-13
    from scipy.linalg import expm
    assert rel(Bl, expm(A * tau) @ B) < 1e-14 and rel(cl, expm(A * tau) @ c) < 1e-14


# --------------------------------------------------------------------- P5 closed form
def test_predict_1d_heat_laplace_closed_form():
    """A=0, l=1: one backward-Euler diffusion step is convolution with the
    Laplace kernel (1/2b) e^{-|y|/b}, b^2 = Q dt/2; on a +-8 sigma periodic grid
    the result is the periodised Gaussian*Laplace (erfc) closed form."""
    N, mu, sig, q, dt = 128, 1.0, 0.5, 1.0, 0.1
    c, B = O.design_grid([mu], [[sig * sig]], (N,), 8.0)
    x = O.grid_points(c, B, (N,))[0]
    g = np.exp(-0.5 * ((x - mu) / sig) ** 2) / (sig * math.sqrt(2 * math.pi))
    wo, _, _ = O.predict_unnormalised(g, c, B, np.zeros((1, 1)), np.array([[q]]), dt, 1)
    b = math.sqrt(0.5 * q * dt)
    L = N * B[0, 0]
    exact = np.zeros(N)
    for m in range(-2, 3):
        y = x - mu + m * L
        exact += (1 / (4 * b)) * np.exp(sig ** 2 / (2 * b * b)) * (
            np.exp(-y / b) * erfc((sig ** 2 / b - y) / (sig * math.sqrt(2)))
            + np.exp(y / b) * erfc((sig ** 2 / b + y) / (sig * math.sqrt(2))))
    assert rel(wo, exact) < 1e-13


# --------------------------------------------------------------------- P6 moments
@pytest.mark.parametrize("case", ["cv2d", "rand3d"])
def test_predict_moments_closed_form(case):
    """The scheme's predicted mean is e^{A tau} m and its covariance the
    Riemann-sum Kalman-Bucy form e^{At}Pe^{A't} + dt sum_n e^{A(t-n dt)} Q
    e^{A'(t-n dt)} (l factors at the start of each substep, R3/R4)."""
    from scipy.linalg import expm
    if case == "cv2d":
        A = np.array([[0.0, 1.0], [0.0, 0.0]])
        Q = np.diag([0.0, 0.1])
        m, P, n, tau, l, ks = np.array([0.3, 1.0]), np.diag([1.0, 0.25]), (96, 96), 0.5, 10, 9.0
    else:
        rng = np.random.default_rng(5)
        A = 0.5 * rng.standard_normal((3, 3))
        Q = 0.3 * np.eye(3) + 0.05 * np.ones((3, 3))
        m, P, n, tau, l, ks = rng.standard_normal(3), np.diag([0.5, 0.3, 0.4]), (40, 40, 40), 0.2, 4, 10.0
    w, c, B = O.initial_density(m, P, n, ks)
    w2, c2, B2 = O.predict(w, c, B, A, Q, tau, l)
    mean, cov = O.moments(w2, c2, B2)
    # the discrete moments of the sampled input (not the continuous P)
    m0, P0 = O.moments(w, c, B)
    F = expm(A * tau)
    dt = tau / l
    covx = F @ P0 @ F.T + dt * sum(expm(A * (tau - s * dt)) @ Q @ expm(A * (tau - s * dt)).T
                                   for s in range(l))
    assert np.max(np.abs(mean - F @ m0)) < 1e-11 * math.sqrt(np.max(np.diag(covx)))
    assert rel(cov, covx) < 1e-10


# --------------------------------------------------------------------- P7, P12, P13
def test_mass_linearity_trace_sign():
    rng = np.random.default_rng(3)
    n = (12, 10)
    A = np.array([[-0.3, 0.8], [0.1, -0.2]])
    Q = np.array([[0.2, 0.05], [0.05, 0.1]])
    B = np.diag([0.2, 0.3])
    c = np.zeros(2)
    u, v = rng.uniform(0, 1, n), rng.uniform(0, 1, n)
    tau, l = 0.3, 5
    wu, _, Bl = O.predict_unnormalised(u, c, B, A, Q, tau, l)
    s = (1 - (tau / l) * np.trace(A)) ** l
    assert abs(wu.sum() - s * u.sum()) < 1e-13 * abs(s * u.sum())          # P7 (DC)
    wv, _, _ = O.predict_unnormalised(v, c, B, A, Q, tau, l)
    wuv, _, _ = O.predict_unnormalised(2.0 * u - 3.0 * v, c, B, A, Q, tau, l)
    assert rel(wuv, 2.0 * wu - 3.0 * wv) < 1e-13                           # P12
    p1, _, _ = O.predict(u, c, B, A, Q, tau, l, trace_sign=O.TRACE_SIGN_PHYSICAL)
    p2, _, _ = O.predict(u, c, B, A, Q, tau, l, trace_sign=O.TRACE_SIGN_PRINTED)
    assert rel(p1, p2) < 1e-14                                              # P13
    assert abs(O.cell_volume(Bl) * p1.sum() - 1.0) < 1e-13


# --------------------------------------------------------------------- P8 KF update
def test_update_conjugate_gaussian_matches_kalman():
    """Gaussian prior x linear-Gaussian likelihood on a SHEARED grid -> the KF
    posterior and the normaliser N(z; Hm, HPH'+R) (eq:filt P:46)."""
    from scipy.linalg import expm
    m = np.array([0.5, -1.0])
    P = np.array([[1.0, 0.3], [0.3, 0.5]])
    c, B0 = O.design_grid(m, P, (128, 128), 10.0)
    A = np.array([[0.0, 1.0], [-0.4, -0.1]])
    F = expm(A * 0.7)
    c, B = F @ c, F @ B0                      # sheared moving grid
    m2, P2 = F @ m, F @ P @ F.T
    X = O.grid_points(c, B, (128, 128))
    w = O.normalise(O.gaussian_pdf(X, m2, P2), B)
    H = np.array([[1.0, 0.5]])
    R = np.array([[0.3]])
    z = np.array([0.9])
    post, logC = O.update(w, c, B, O.lik_linear_gauss(X, z, H, R))
    mean, cov = O.moments(post, c, B)
    S = H @ P2 @ H.T + R
    K = P2 @ H.T @ np.linalg.inv(S)
    mk = m2 + K @ (z - H @ m2)
    Pk = (np.eye(2) - K @ H) @ P2
    r = z - H @ m2
    logZ = -0.5 * float(r @ np.linalg.solve(S, r)) - 0.5 * math.log(2 * math.pi * np.linalg.det(S))
    assert np.max(np.abs(mean - mk)) < 1e-12
    assert rel(cov, Pk) < 1e-11
    assert abs(logC - logZ) < 1e-12


def test_range_likelihood_reduces_to_linear_for_positive_x():
    X = np.linspace(0.1, 3.0, 50).reshape(1, -1)
    a = O.lik_range_gauss(X, [1.2], 0.3)
    b = O.lik_linear_gauss(X, [1.2], [[1.0]], [[0.09]])
    assert rel(a, b) < 1e-14
    zz = np.linspace(-10, 10, 20001)
    # int p(z|x) dz = 1 for fixed x (quadrature on a wide z grid)
    vals = np.array([O.lik_range_gauss(np.array([[0.4], [0.3]]), [z_], 0.5)[0] for z_ in zz])
    assert abs(np.trapezoid(vals, zz) - 1.0) < 1e-10


# --------------------------------------------------------------------- P10 regrid
def test_regrid_identity_and_affine():
    rng = np.random.default_rng(4)
    n = (10, 8)
    c = np.array([0.2, -0.1])
    B = np.array([[0.3, 0.05], [-0.02, 0.25]])
    w = rng.uniform(0.1, 1.0, n)
    assert rel(O.interpolate(w, c, B, O.grid_points(c, B, n)), w) < 1e-15
    # affine data is reproduced exactly by multilinear interpolation inside the support
    U = np.stack(np.meshgrid(O.axis_offsets(10), O.axis_offsets(8), indexing="ij"))
    aff = 2.0 + 0.3 * U[0] - 0.7 * U[1]
    cn = c + B @ np.array([0.5, -0.25])          # shift by a fraction of a cell
    Xn = O.grid_points(cn, B, n)
    vals = O.interpolate(aff, c, B, Xn)
    Un = U + np.array([0.5, -0.25]).reshape(2, 1, 1)
    inside = (Un[0] <= 4.5) & (Un[0] >= -4.5) & (Un[1] >= -3.5) & (Un[1] <= 3.5)
    exact = 2.0 + 0.3 * Un[0] - 0.7 * Un[1]
    assert np.max(np.abs(vals[inside] - exact[inside])) < 1e-14
    # zero ghost nodes: half a cell outside the first node gives half its value
    one = O.interpolate(np.ones((4,)), np.zeros(1), np.eye(1), np.array([[-2.0, -2.5, -1.75]]))
    assert np.allclose(one, [0.5, 0.0, 0.75], atol=1e-15)


# --------------------------------------------------------------------- P11 symmetry
def test_symmetry():
    n = (16, 12)
    w, c, B = O.initial_density([0.0, 0.0], np.diag([1.0, 0.5]), n, 6.0)
    w2, c2, B2 = O.predict(w, c, B, np.zeros((2, 2)), np.diag([0.3, 0.2]), 0.5, 5)
    assert np.max(np.abs(w2 - w2[::-1, ::-1])) < 1e-15 * np.max(w2) * 10
    mean, _ = O.moments(w2, c2, B2)
    assert np.max(np.abs(mean)) < 1e-15


# --------------------------------------------------------------------- grid / normalise goldens
def test_grid_and_normalise_goldens():
    g = GOLD["build_grid"]
    c, B = O.design_grid([0.0], [[g["sigma"] ** 2]], (g["N"],), g["k_sigma"])
    assert np.allclose(O.grid_points(c, B, (g["N"],))[0], g["expected_points"], atol=1e-15)
    g = GOLD["normalise_uniform"]
    w = O.normalise(np.ones(g["N"]), np.array([[g["delta"]]]))
    assert np.allclose(w, g["expected"], atol=1e-15)


def test_moments_gaussian():
    """N(0,1) on +-5 sigma, N=128 -> variance within 1%; on a wide
    grid the midpoint rule is spectrally accurate."""
    w, c, B = O.initial_density([0.0], [[1.0]], (128,), 5.0)
    _, cov = O.moments(w, c, B)
    assert abs(cov[0, 0] - 1.0) < 0.01
    m = np.array([0.3, -0.2])
    P = np.array([[0.8, 0.2], [0.2, 0.4]])
    w, c, B = O.initial_density(m, P, (64, 64), 9.0)
    mean, cov = O.moments(w, c, B)
    assert np.max(np.abs(mean - m)) < 1e-13 and rel(cov, P) < 1e-12


# --------------------------------------------------------------------- P9 whole filter
@pytest.mark.slow
def test_filter_converges_to_kalman_first_order_in_dt():
    """Linear-Gaussian 1-D (C1 model) whole filter vs the continuous-discrete
    KF: error is O(dt) (backward Euler), so l=10 -> l=100 shrinks it ~10x."""
    from workloads import make_config, simulate
    from scipy.linalg import expm
    errs = []
    for l in (10, 100):
        cfg = make_config("C1", n=(256,), k_sigma=8.0, l=l, T=10)
        zs = simulate(cfg)["z"]
        rec = O.run_filter(cfg, zs)
        # KF
        a, q = cfg.A[0, 0], cfg.Q[0, 0]
        F = math.exp(a * cfg.tau)
        Qd = q * (math.exp(2 * a * cfg.tau) - 1) / (2 * a)
        m, P = cfg.prior_mean[0, 0], cfg.prior_cov[0, 0]
        e = 0.0
        for k in range(cfg.T + 1):
            if k:
                m, P = F * m, F * P * F + Qd
            S = P + cfg.R[0, 0]
            K = P / S
            m, P = m + K * (zs[k, 0, 0] - m), (1 - K) * P
            e = max(e, abs(rec["mean"][k][0] - m) / math.sqrt(P))
        errs.append(e)
    assert errs[0] / errs[1] > 5.0, errs

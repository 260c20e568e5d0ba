"""CPU ORACLE for the spectral point-mass filter -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this module. The product path
(``paper_2412_07240_b200``) never imports it, and it imports nothing from the
product: the two share no code (the seeded input generator ``workloads`` holds
no method arithmetic).

Plain, slow, obviously-correct fp64 numpy, written step by step from
/root/reference/PAPER.md (cited as ``P:<line>``) with the readings R1-R22 of
SURVEY.md §8(c) (restated in DESIGN.md §3) wherever the paper is silent or
garbled:

* the DFT is the O(N^2) definition eq:fourtrsf, a dense N x N matrix
  applied along each axis in turn (Alg. 1) -- no FFT;
* the spectral multiplier is the full tensor Psi over ALL N^nx wavenumbers
  (no half-spectrum / Hermitian packing, which the CUDA path uses);
* normalisation is by explicit summation (Alg. 6), not the closed form;
* moments are accumulated in PHYSICAL coordinates (the CUDA path uses index
  coordinates and maps back).

Array convention: a density on an ``n = (N_0, ..., N_{nx-1})`` grid is an array
of shape ``n`` indexed ``w[j_0, j_1, ...]``. The library's memory layout (axis 0
fastest, P:114 MATLAB-style reshape) is ``w.transpose(reversed axes)`` -- see
``to_lib`` / ``from_lib``.

Parity status of each function is stated in its docstring ("pinned by" the
tests that fix it independently of this code, or "parity unpinned").
"""
from __future__ import annotations

import itertools
import math

import numpy as np
from scipy.linalg import expm as _scipy_expm

TRACE_SIGN_PHYSICAL = -1   # R5: s = (1 - dt tr A)^l  (eq:easyFPE P:92, b_t P:164)
TRACE_SIGN_PRINTED = +1    # Alg. 4 as printed: (1 + dt tr A)^l
DIFF_FULL = 0              # R3: D_n = B_n^{-1} Q B_n^{-T} with cross terms
DIFF_AXIS_LITERAL = 1      # Alg. 2/3 literally: per-axis L^(m), no cross terms
DIFF_FDM = 2               # NEXT-1: the paper's FDM baseline (eq:FDM), in its FST form (eq:FST)
STEP_EULER = 0             # the paper's semi-implicit Euler substeps (Alg. 3)
STEP_CN = 1                # NEXT-4: Crank-Nicolson substeps ("higher order time stepping"; R27)
GRID_AXIS = 0              # R12: grids designed axis-aligned from a covariance
GRID_EIGEN = 1             # R28 (NEXT-4): grids aligned with the covariance eigenvectors (refs of P:346)


class NoSupportError(RuntimeError):
    """Measurement incompatible with the grid support (normaliser 0/non-finite)."""


# ----------------------------------------------------------------------------
# layout helpers (not method arithmetic)
# ----------------------------------------------------------------------------
def to_lib(w: np.ndarray) -> np.ndarray:
    """logical [j0, j1, ...] -> library layout (axis 0 fastest, C order)."""
    return np.ascontiguousarray(w.transpose(tuple(reversed(range(w.ndim)))))


def from_lib(w: np.ndarray, n: tuple) -> np.ndarray:
    """library layout (..., N_1, N_0) -> logical [j0, j1, ...]."""
    a = np.asarray(w).reshape(tuple(reversed(n)))
    return a.transpose(tuple(reversed(range(len(n)))))


# ----------------------------------------------------------------------------
# grid and point-mass density
# ----------------------------------------------------------------------------
def axis_offsets(N: int) -> np.ndarray:
    """Cell-centred index offsets u_j = j - (N-1)/2, j = 0..N-1 (R10; the grid
    size is L = N delta). Pinned by test_grid (symmetry, spacing)."""
    return np.arange(N, dtype=np.float64) - (N - 1) / 2.0


def design_grid(mean, cov, n, k_sigma):
    """Axis-aligned grid centred at ``mean`` spanning +-k_sigma std per axis:
    c = mean, B = diag(2 k_sigma sqrt(cov_mm) / N_m) (R10; paper silent, its
    L_t = N delta_t P:219). Pinned by test_grid."""
    mean = np.asarray(mean, dtype=np.float64)
    cov = np.asarray(cov, dtype=np.float64)
    d = np.array([2.0 * k_sigma * math.sqrt(cov[m, m]) / n[m] for m in range(len(n))])
    return mean.copy(), np.diag(d)


def grid_points(c, B, n) -> np.ndarray:
    """Physical points xi = c + B u for all multi-indices; shape (nx, *n).
    P:114 (grid xi_t), footnote P:121 (equidistant), R-layout."""
    U = np.stack(np.meshgrid(*[axis_offsets(N) for N in n], indexing="ij"))
    return np.asarray(c).reshape((-1,) + (1,) * len(n)) + np.tensordot(B, U, axes=(1, 0))


def cell_volume(B) -> float:
    """Volume of a point's neighbourhood, |det B| (P:120 'delta_t is the
    volume', footnote P:121; R9)."""
    return abs(float(np.linalg.det(np.asarray(B, dtype=np.float64))))


def normalise(w, B) -> np.ndarray:
    """P = P~ / (vol sum P~)  (P:120 with the garbled c_t read as R9).
    Pinned by test_normalise (SPEC S:168 example)."""
    tot = cell_volume(B) * float(np.sum(w))
    if not np.isfinite(tot) or tot == 0.0:
        raise NoSupportError("normaliser is zero or non-finite")
    return w / tot


def gaussian_pdf(X, m, P) -> np.ndarray:
    """N(x; m, P) at points X (nx, ...)."""
    m = np.asarray(m, dtype=np.float64)
    P = np.asarray(P, dtype=np.float64)
    nx = m.shape[0]
    d = X - m.reshape((-1,) + (1,) * (X.ndim - 1))
    Pi = np.linalg.inv(P)
    e = np.einsum("a...,ab,b...->...", d, Pi, d)
    return np.exp(-0.5 * e) / math.sqrt((2 * math.pi) ** nx * np.linalg.det(P))


def eigen_grid(mean, cov, n, k_sigma):
    """R28 (the covariance-aligned grids of the refs of P:346):
    c = mean, B's columns along the eigenvectors of cov, each spanning
    +-k_sigma sqrt(lambda): cov = V diag(lambda) V^T (LAPACK symmetric eigensolver);
    eigenvector j in order of decreasing lambda (lower index first on ties) takes the
    still free axis a of its largest |V[a, j]| (lowest axis on ties), with the sign
    that makes V[a, j] > 0; B[:, a] = v_j 2 k_sigma sqrt(lambda_j) / N_a.
    Pinned by test_oracle_eigen_grid (B diag(N) (B diag(N))^T = 4 k_sigma^2 cov;
    diagonal cov -> design_grid; a known rotation)."""
    mean = np.asarray(mean, dtype=np.float64)
    cov = np.asarray(cov, dtype=np.float64)
    nx = len(n)
    lam, V = np.linalg.eigh(0.5 * (cov + cov.T))
    if not np.all(np.isfinite(lam)) or np.any(lam <= 0.0):
        raise NoSupportError("covariance not positive definite: cannot design grid")
    order = sorted(range(nx), key=lambda j: (-lam[j], j))
    free = list(range(nx))
    B = np.zeros((nx, nx))
    for j in order:
        a = max(free, key=lambda k: (abs(V[k, j]), -k))
        free.remove(a)
        v = V[:, j] if V[a, j] > 0.0 else -V[:, j]
        B[:, a] = v * 2.0 * k_sigma * math.sqrt(lam[j]) / n[a]
    return mean.copy(), B


def grid_design(mean, cov, n, k_sigma, grid=GRID_AXIS):
    """The grid a covariance designs: R12/R10 axis-aligned or R28 eigen-aligned."""
    if grid == GRID_EIGEN:
        return eigen_grid(mean, cov, n, k_sigma)
    return design_grid(mean, cov, n, k_sigma)


def initial_density(mean, cov, n, k_sigma, grid=GRID_AXIS):
    """p(x_0) sampled on the designed grid and normalised (P:48 footnote:
    the first predictive PDF is p(x_0)). Returns (w, c, B)."""
    c, B = grid_design(mean, cov, n, k_sigma, grid)
    w = gaussian_pdf(grid_points(c, B, n), mean, cov)
    return normalise(w, B), c, B


# ----------------------------------------------------------------------------
# spectral differentiation
# ----------------------------------------------------------------------------
def dft_matrix(N: int, inverse: bool = False) -> np.ndarray:
    """eq:fourtrsf: P^(s) = (1/N) sum_j P^(j) exp(-2 pi i j s / N).
    Forward carries the 1/N, the inverse (P:233, P:239 'sum_s ... exp(+...)')
    is unscaled (R6). Angles use (j s mod N) to avoid large arguments."""
    j = np.arange(N)
    ang = 2.0 * math.pi * ((np.outer(j, j) % N).astype(np.float64)) / N
    if inverse:
        return np.cos(ang) + 1j * np.sin(ang)                 # [j, s]
    return (np.cos(ang) - 1j * np.sin(ang)) / N               # [s, j]


def dft_axis(a: np.ndarray, axis: int, inverse: bool = False) -> np.ndarray:
    """Apply the dense 1-D DFT matrix along one axis (naive O(N^2) per line)."""
    F = dft_matrix(a.shape[axis], inverse)
    out = np.tensordot(F, a, axes=([1], [axis]))
    return np.moveaxis(out, 0, axis)


def dftn(w: np.ndarray) -> np.ndarray:
    """Alg. 1: transform 'dimension by dimension'."""
    S = w.astype(np.complex128)
    for ax in range(w.ndim):
        S = dft_axis(S, ax, inverse=False)
    return S


def idftn(S: np.ndarray) -> np.ndarray:
    """Alg. 5: inverse transform dimension by dimension, unscaled."""
    for ax in range(S.ndim):
        S = dft_axis(S, ax, inverse=True)
    return S


def wavenumbers(N: int) -> np.ndarray:
    """Integer wavenumbers in transform order, fftshift(-N/2 : N/2-1) (P:310,
    Alg. 2): [0, 1, ..., N/2-1, -N/2, ..., -1]. N must be even."""
    if N % 2:
        raise ValueError("N must be even (P:219)")
    return np.concatenate([np.arange(0, N // 2), np.arange(-N // 2, 0)]).astype(np.float64)


def second_derivative_coeffs(N: int, L: float) -> np.ndarray:
    """c'' = -(2 pi / L * fftshift(-N/2:N/2-1))^2  (Alg. 2).
    Pinned by the SPEC S:412 golden (N=4, L=2pi -> -[0,1,4,1])."""
    return -((2.0 * math.pi / L) * wavenumbers(N)) ** 2


def spectral_second_derivative(p: np.ndarray, L: float) -> np.ndarray:
    """1-D p'' at the grid points via eq:secDer: multiply the DFT
    by c'' (Nyquist term kept) and invert. Pinned by exactness on
    band-limited modes (test_spectral)."""
    S = dft_axis(p.astype(np.complex128), 0) * second_derivative_coeffs(p.shape[0], L)
    return dft_axis(S, 0, inverse=True).real


def spectral_first_derivative(p: np.ndarray, L: float) -> np.ndarray:
    """1-D p' via P:230-234: multiplier 2 pi i s / L over 0<|s|<N/2, the Nyquist
    term dropped (the sum is over 0<s<N/2; R7/R8 signed-k reading)."""
    N = p.shape[0]
    k = wavenumbers(N)
    mult = 1j * (2.0 * math.pi / L) * k
    mult[N // 2] = 0.0
    S = dft_axis(p.astype(np.complex128), 0) * mult
    return dft_axis(S, 0, inverse=True).real


# ----------------------------------------------------------------------------
# FPE time update: moving grid + spectral semi-implicit Euler (§V)
# ----------------------------------------------------------------------------
def expm(M) -> np.ndarray:
    """Matrix exponential (library primitive); grid motion xi' = A xi (P:82,
    eq:gridMov P:142, delta_n = e^{A dt} delta_{n-1} P:148)."""
    return _scipy_expm(np.asarray(M, dtype=np.float64))


def index_diffusion(Bn, Q, mode: int = DIFF_FULL) -> np.ndarray:
    """Diffusion matrix of (1/2) div(Q grad p) (eq:easyFPE P:93) written in the
    moving grid's index coordinates u = B_n^{-1}(x - c_n).

    DIFF_FULL (R3): D_n = B_n^{-1} Q B_n^{-T} (cross terms kept). For a diagonal
    B_n = diag(delta_m) it reduces to D_mm = Q_mm / delta_m^2, i.e. exactly Alg.
    3's -c''_m Q_mm with L^(m) = N delta_m.
    DIFF_AXIS_LITERAL: Alg. 2/3 literally -- D_mm = Q_mm / delta_m^2 with
    delta_m the length of B_n's m-th column (L^(m) = N delta_m), no
    cross terms."""
    Bn = np.asarray(Bn, dtype=np.float64)
    Q = np.asarray(Q, dtype=np.float64)
    if mode == DIFF_FULL:
        Bi = np.linalg.inv(Bn)
        return Bi @ Q @ Bi.T
    delta = np.linalg.norm(Bn, axis=0)
    return np.diag(np.diag(Q) / delta ** 2)


def psi_factor(D: np.ndarray, dt: float, n: tuple) -> np.ndarray:
    """One Euler factor psi_n over the full wavenumber grid (Alg. 3 P:333-336,
    Euler display P:313-318 read as R2):

        psi = 1 / (1 + dt/2 q),   q = quad_form(D, n)
            = 1 / (1 + dt/2 [ sum_m D_mm kappa_m^2 + 2 sum_{m<m'} D_mm' kx_m kx_m' ])

    kappa_m = 2 pi k_m / N_m (index coordinates, so -c''_m Q_mm = D_mm kappa_m^2
    on a diagonal grid); kx is kappa with the Nyquist wavenumber zeroed (R7: the
    first-derivative symbol drops Nyquist), the squared terms keep it
    (P:238). Pinned by test_spectral (S:440 golden, 0 < psi <= 1, psi(0) = 1)
    and the dense brute-force solve (P4); the symbol itself is quad_form's (one copy,
    shared with the Crank-Nicolson factors)."""
    return 1.0 / (1.0 + 0.5 * dt * quad_form(D, n))


def trace_factor(A, dt: float, l: int, sign: int = TRACE_SIGN_PHYSICAL) -> float:
    """s = (1 + sign dt trace(A))^l (Alg. 4; sign per R5). The base must be
    positive (an Euler factor <= 0 is a step-size error)."""
    base = 1.0 + sign * dt * float(np.trace(np.asarray(A)))
    if base <= 0.0:
        raise ValueError("1 -/+ dt tr(A) <= 0: Euler step too large")
    return base ** l


def quad_form(D: np.ndarray, n: tuple) -> np.ndarray:
    """q(k) = sum_m D_mm kappa_m^2 + 2 sum_{m<m'} D_mm' kx_m kx_m' over the full
    wavenumber grid (kappa = 2 pi k / N, kx = kappa with Nyquist zeroed, R7): the symbol of
    -div(D grad) in index coordinates, so psi_factor = 1 / (1 + dt/2 q)."""
    nx = len(n)
    kap, kapx = [], []
    for m, N in enumerate(n):
        k = 2.0 * math.pi * wavenumbers(N) / N
        kx = k.copy()
        kx[N // 2] = 0.0
        shape = [1] * nx
        shape[m] = N
        kap.append(k.reshape(shape))
        kapx.append(kx.reshape(shape))
    q = np.zeros(n)
    for a in range(nx):
        q = q + D[a, a] * kap[a] ** 2
        for b in range(a + 1, nx):
            q = q + 2.0 * D[a, b] * kapx[a] * kapx[b]
    return q


def predict_unnormalised(w, c, B, A, Q, tau, l, diff_mode=DIFF_FULL,
                         trace_sign=TRACE_SIGN_PHYSICAL, step=STEP_EULER):
    """Alg. 1-5 over one prediction interval tau with l Euler
    substeps dt = tau/l.

    1. S = DFT of the weights, dimension by dimension (1/N per axis).
    2-3. Psi = prod_{n=0}^{l-1} psi_n, psi_n built from the diffusion in the
       grid's index coordinates at the START of substep n, B_n = e^{A n dt} B
       (R4: l factors; R3).
    4. S <- Psi (.) S (1 -/+ dt tr A)^l.
    5. inverse DFT; the result is real (Psi is even) -- the imaginary residue is
       checked and dropped.
    The grid moves with the drift: c <- e^{A tau} c, B <- e^{A tau} B.
    Returns (w_unnormalised, c_l, B_l)."""
    n = w.shape
    dt = tau / l
    S = dftn(w)
    Psi = np.ones(n)
    if step == STEP_CN:
        # R27 Crank-Nicolson for the diffusion d P/dt = -(1/2) q(t) P per wavenumber, with the
        # moving grid's time-dependent q: P_{n+1} (1 + dt/4 q_{n+1}) = P_n (1 - dt/4 q_n),
        # q_n on the grid at t_n = n dt (l + 1 grids); second order in dt
        for s_ in range(l):
            qa = quad_form(index_diffusion(expm(np.asarray(A) * (s_ * dt)) @ B, Q, diff_mode), n)
            qb = quad_form(index_diffusion(expm(np.asarray(A) * ((s_ + 1) * dt)) @ B, Q, diff_mode), n)
            Psi = Psi * (1.0 - 0.25 * dt * qa) / (1.0 + 0.25 * dt * qb)
    for s_ in range(l if step == STEP_EULER else 0):
        Bn = expm(np.asarray(A) * (s_ * dt)) @ B
        Psi = Psi * psi_factor(index_diffusion(Bn, Q, diff_mode), dt, n)
    S = S * (Psi * trace_factor(A, dt, l, trace_sign))
    out = idftn(S)
    scale = max(float(np.max(np.abs(out.real))), 1e-300)
    if float(np.max(np.abs(out.imag))) > 1e-9 * scale:
        raise AssertionError("inverse transform is not real: symbol not even?")
    M = expm(np.asarray(A) * tau)
    return out.real.copy(), M @ np.asarray(c), M @ np.asarray(B)


def predict(w, c, B, A, Q, tau, l, diff_mode=DIFF_FULL, trace_sign=TRACE_SIGN_PHYSICAL, step=STEP_EULER):
    """Alg. 1-6: the unnormalised update followed by normalisation by explicit
    summation on the moved grid (Alg. 6, R9). Returns (w, c_l, B_l).
    diff_mode DIFF_FDM: the FDM baseline in its FST form (eq:FST), same normalisation."""
    if diff_mode == DIFF_FDM:
        wu, cl, Bl = fst_predict_unnormalised(w, c, B, A, Q, tau, l, trace_sign)
    else:
        wu, cl, Bl = predict_unnormalised(w, c, B, A, Q, tau, l, diff_mode, trace_sign, step)
    return normalise(wu, Bl), cl, Bl


# ----------------------------------------------------------------------------
# NEXT-1 baseline: explicit finite differences (eq:FDM P:144-150) and their
# eigenvalue / fast-sine-transform form (eq:fdiff P:158-164, eq:FKEnumSol P:167-170,
# P:178-196, eq:FST P:199-202). Readings: R23 l factors (n = 0..l-1,
# as R4) although eq:FKEnumSol prints l+1; R24 zero Dirichlet boundary (F_diff is the
# finite tridiagonal matrix, rows truncated at the grid edge); R25 multi-D = one
# central difference per axis with that axis's spacing delta_m = ||B_n[:, m]|| and
# Q_mm, the trace term (1 - dt tr A) per step (b_t P:164, physical sign R5).
# ----------------------------------------------------------------------------
def fdm_axis_spacing(Bn) -> np.ndarray:
    """delta_m of the moving grid: length of B_n's m-th column (1-D: delta_n =
    e^{A dt} delta_{n-1})."""
    return np.linalg.norm(np.asarray(Bn, dtype=np.float64), axis=0)


def fdm_matrix(N: int, a: float, b: float) -> np.ndarray:
    """F_diff (eq:fdiff P:158-162): tridiagonal Toeplitz, b on the diagonal, a on
    both off-diagonals, zero Dirichlet boundary (R24). Pinned by the closed-form
    eigenvalues and by fst == fdm."""
    return b * np.eye(N) + a * (np.eye(N, k=1) + np.eye(N, k=-1))


def fdm_step_coeffs(Bn, A, Q, dt, sign: int = TRACE_SIGN_PHYSICAL):
    """Per axis a_m = Q_mm dt / (2 delta_m^2) and the diagonal b =
    1 + sign dt tr(A) - sum_m 2 a_m (b_t P:164; R5, R25)."""
    delta = fdm_axis_spacing(Bn)
    a = np.diag(np.asarray(Q, dtype=np.float64)) * dt / (2.0 * delta ** 2)
    b = 1.0 + sign * dt * float(np.trace(np.asarray(A))) - 2.0 * float(np.sum(a))
    return a, b


def fdm_predict_unnormalised(w, c, B, A, Q, tau, l, trace_sign=TRACE_SIGN_PHYSICAL):
    """eq:FDM literally: l explicit steps P_{n+1} = F_n P_n with the central
    difference along every axis,
        F_n P = b_n P + sum_m a_{m,n} (P shifted +1 along m + P shifted -1 along m),
    zero outside the grid (R24), coefficients on the grid at the start of step n,
    B_n = e^{A n dt} B (R23). Each shift-sum is the dense off-diagonal part of F_diff
    applied along axis m. The grid moves with the drift (eq:gridMov P:142)."""
    w = np.asarray(w, dtype=np.float64)
    n = w.shape
    dt = tau / l
    P = w.copy()
    for s_ in range(l):
        Bn = expm(np.asarray(A) * (s_ * dt)) @ B
        a, b = fdm_step_coeffs(Bn, A, Q, dt, trace_sign)
        out = b * P
        for m in range(len(n)):
            off = fdm_matrix(n[m], 1.0, 0.0)                  # the a-pattern of F_diff, unit weight
            out = out + a[m] * np.moveaxis(np.tensordot(off, np.moveaxis(P, m, 0), axes=(1, 0)), 0, m)
        P = out
    M = expm(np.asarray(A) * tau)
    return P, M @ np.asarray(c), M @ np.asarray(B)


def dst1_matrix(N: int) -> np.ndarray:
    """Eigenvector matrix R of F_diff, R[j, i] = sin((i+1)(j+1) pi/(N+1));
    R^{-1} = 2/(N+1) R. Pinned by the orthogonality test."""
    j = np.arange(1, N + 1)
    return np.sin(np.outer(j, j) * math.pi / (N + 1))


def fdm_eigenvalues(N: int, a: float, b: float) -> np.ndarray:
    """lambda^{(j-1)} = b + 2a cos(j pi/(N+1)), j = 1..N. Pinned against a
    library eigensolver."""
    j = np.arange(1, N + 1)
    return b + 2.0 * a * np.cos(j * math.pi / (N + 1))


def fst_predict_unnormalised(w, c, B, A, Q, tau, l, trace_sign=TRACE_SIGN_PHYSICAL):
    """eq:FST, multi-D: sine transform along every axis (R_m applied along
    axis m), multiply by Lambda = prod_{n<l} lambda_n with the eigenvalue of the
    per-step operator at multi-index j,
        lambda_n(j) = b_n + sum_m 2 a_{m,n} cos((j_m+1) pi/(N_m+1))
    (the axes' difference operators share the DST eigenvectors), inverse transform
    R^{-1} = 2/(N_m+1) R_m per axis. Equal to fdm_predict_unnormalised
    (T_k = R Lambda R^{-1})."""
    w = np.asarray(w, dtype=np.float64)
    n = w.shape
    nx = len(n)
    dt = tau / l
    S = w.copy()
    for m in range(nx):
        S = np.moveaxis(np.tensordot(dst1_matrix(n[m]), np.moveaxis(S, m, 0), axes=(1, 0)), 0, m)
    Lam = np.ones(n)
    for s_ in range(l):
        Bn = expm(np.asarray(A) * (s_ * dt)) @ B
        a, b = fdm_step_coeffs(Bn, A, Q, dt, trace_sign)
        lam = np.full(n, b)
        for m in range(nx):
            shape = [1] * nx
            shape[m] = n[m]
            lam = lam + (fdm_eigenvalues(n[m], a[m], 0.0)).reshape(shape)
        Lam = Lam * lam
    S = S * Lam
    for m in range(nx):
        R = dst1_matrix(n[m]) * (2.0 / (n[m] + 1))
        S = np.moveaxis(np.tensordot(R, np.moveaxis(S, m, 0), axes=(1, 0)), 0, m)
    M = expm(np.asarray(A) * tau)
    return S, M @ np.asarray(c), M @ np.asarray(B)


# ----------------------------------------------------------------------------
# measurement update and moments
# ----------------------------------------------------------------------------
def lik_linear_gauss(X, z, H, R) -> np.ndarray:
    """p(z | x) for z = H x + v, v ~ N(0, R) (eq:meas P:36) at points X
    (R13: full Gaussian constant)."""
    H = np.asarray(H, dtype=np.float64)
    R = np.asarray(R, dtype=np.float64)
    z = np.asarray(z, dtype=np.float64).reshape(-1)
    nz = H.shape[0]
    r = z.reshape((-1,) + (1,) * (X.ndim - 1)) - np.tensordot(H, X, axes=(1, 0))
    e = np.einsum("a...,ab,b...->...", r, np.linalg.inv(R), r)
    return np.exp(-0.5 * e) / math.sqrt((2 * math.pi) ** nz * np.linalg.det(R))


def lik_range_gauss(X, z, sigma) -> np.ndarray:
    """p(z | x) for z = ||x|| + v, v ~ N(0, sigma^2) (C3's h; eq:meas P:36)."""
    rng = np.sqrt(np.sum(X * X, axis=0))
    z = float(np.asarray(z).reshape(-1)[0])
    return np.exp(-0.5 * ((z - rng) / sigma) ** 2) / (sigma * math.sqrt(2 * math.pi))


def terrain_height(px, py, heights, x0, y0, dx, dy):
    """The map h of the paper's §VI measurement ("a table function that assigns
    vertical position to each combination of latitude and longitude it covers"): bilinear
    between the table nodes heights[r, c] at (x0 + c dx, y0 + r dy), the nearest edge value
    outside the table (R26). Pinned by exactness on bilinear fields and the node values."""
    H = np.asarray(heights, dtype=np.float64)
    nrow, ncol = H.shape
    u = np.clip((np.asarray(px, dtype=np.float64) - x0) / dx, 0.0, ncol - 1)
    v = np.clip((np.asarray(py, dtype=np.float64) - y0) / dy, 0.0, nrow - 1)
    c = np.minimum(np.floor(u).astype(np.int64), ncol - 2)
    r = np.minimum(np.floor(v).astype(np.int64), nrow - 2)
    fu, fv = u - c, v - r
    return ((1 - fu) * (1 - fv) * H[r, c] + fu * (1 - fv) * H[r, c + 1]
            + (1 - fu) * fv * H[r + 1, c] + fu * fv * H[r + 1, c + 1])


def lik_terrain_gm(X, z, table, gm) -> np.ndarray:
    """p(z | x) for z = h(x_ix, x_iy) + v with the 2-component (here: any) Gaussian-mixture
    noise of eq:ex1_PDF: sum_g w_g N(z - h; mu_g, var_g), weights normalised.
    ``table`` = (heights, x0, y0, dx, dy, ix, iy); ``gm`` = ((w, mu, var), ...)."""
    heights, x0, y0, dx, dy, ix, iy = table
    d = float(np.asarray(z).reshape(-1)[0]) - terrain_height(X[ix], X[iy], heights, x0, y0, dx, dy)
    wsum = sum(g[0] for g in gm)
    out = np.zeros_like(d)
    for w, mu, var in gm:
        out = out + (w / wsum) * np.exp(-0.5 * (d - mu) ** 2 / var) / math.sqrt(2 * math.pi * var)
    return out


def update(w, c, B, lik_values):
    """Bayes' rule eq:filt: posterior = prior x likelihood / normaliser,
    normaliser p(z_k|z^{k-1}) = int prior x lik dx by quadrature over
    the point-mass cells, vol sum w_i lik_i. Returns (posterior, log normaliser).
    Pinned by the conjugate-Gaussian KF closed form (P8)."""
    prod = w * lik_values
    C = cell_volume(B) * float(np.sum(prod))
    if not np.isfinite(C) or C <= 0.0:
        raise NoSupportError("measurement incompatible with grid support")
    return prod / C, math.log(C)


def moments(w, c, B):
    """Mean and covariance of the point-mass density (first two moments, P:75;
    E[x|z], var P:434; R14 population moments, symmetrised), accumulated
    directly in PHYSICAL coordinates: mean = vol sum xi w, cov = vol sum
    (xi-mean)(xi-mean)^T w. Pinned by P8 (KF) and P6 (closed-form predict)."""
    n = w.shape
    X = grid_points(c, B, n)
    vol = cell_volume(B)
    mass = vol * float(np.sum(w))
    nx = len(n)
    mean = np.array([vol * float(np.sum(X[a] * w)) for a in range(nx)]) / mass
    d = X - mean.reshape((-1,) + (1,) * nx)
    cov = np.empty((nx, nx))
    for a in range(nx):
        for b in range(nx):
            cov[a, b] = vol * float(np.sum(d[a] * d[b] * w)) / mass
    return mean, 0.5 * (cov + cov.T)


# ----------------------------------------------------------------------------
# re-centring the grid (paper silent; north_star "re-centre the grid"; R12)
# ----------------------------------------------------------------------------
def regrid_target(mean, cov, n, k_sigma, grid=GRID_AXIS):
    """New grid at the posterior mean: axis-aligned, +-k_sigma sqrt(cov_mm) (R12), or
    eigen-aligned (R28, eigen_grid). parity unpinned (policy invented; SURVEY
    'Parity unpinned')."""
    cov = np.asarray(cov)
    if any((not np.isfinite(cov[m, m])) or cov[m, m] <= 0.0 for m in range(len(n))):
        raise NoSupportError("degenerate covariance: cannot design grid")
    return grid_design(mean, cov, n, k_sigma, grid)


def interpolate(w, c, B, X) -> np.ndarray:
    """Multilinear interpolation of the weights w (grid c, B) at physical points
    X (nx, ...): fractional old index v = B^{-1}(x - c) + (N-1)/2 per axis,
    2^nx surrounding nodes, nodes outside 0..N-1 count as zero (zero ghost
    nodes, R12). Pinned by P10 (identity, affine exactness)."""
    n = w.shape
    nx = len(n)
    Bi = np.linalg.inv(np.asarray(B))
    d = X - np.asarray(c).reshape((-1,) + (1,) * (X.ndim - 1))
    V = np.tensordot(Bi, d, axes=(1, 0))
    for m in range(nx):
        V[m] += (n[m] - 1) / 2.0
    i0 = np.floor(V)
    f = V - i0
    i0 = i0.astype(np.int64)
    out = np.zeros(X.shape[1:])
    for corner in itertools.product((0, 1), repeat=nx):
        wt = np.ones(X.shape[1:])
        idx = []
        ok = np.ones(X.shape[1:], dtype=bool)
        for m in range(nx):
            im = i0[m] + corner[m]
            wt = wt * (f[m] if corner[m] else (1.0 - f[m]))
            ok &= (im >= 0) & (im <= n[m] - 1)
            idx.append(np.clip(im, 0, n[m] - 1))
        out = out + wt * np.where(ok, w[tuple(idx)], 0.0)
    return out


def regrid(w, c, B, c_new, B_new):
    """Resample onto the new grid and renormalise by summation (R12)."""
    Xn = grid_points(c_new, B_new, w.shape)
    return normalise(interpolate(w, c, B, Xn), B_new)


# ----------------------------------------------------------------------------
# one filter run (R15: update at k=0 on the prior, then T x (predict, update))
# ----------------------------------------------------------------------------
def make_likelihood(cfg, X, z):
    if cfg.lik_kind == 1:
        return lik_range_gauss(X, z, cfg.sigma)
    if cfg.lik_kind == 2:
        from workloads import terrain_table      # the map is an input (seeded synthetic field)
        return lik_terrain_gm(X, z, terrain_table(cfg), cfg.extra["gm"])
    return lik_linear_gauss(X, z, cfg.H, cfg.R)


def run_filter(cfg, zs, b: int = 0, T: int | None = None, keep_weights: bool = False,
               diff_mode: int = DIFF_FULL, trace_sign: int = TRACE_SIGN_PHYSICAL, step: int = STEP_EULER,
               grid: int = GRID_AXIS):
    """Run filter ``b`` of config ``cfg`` on measurements ``zs`` (T+1, batch, nz).

    Epoch k: [k>0: predict(tau, l)] -> update(z_k) -> moments -> regrid.
    Records per epoch the moments, log normaliser, the posterior grid and
    (optionally) the posterior weights before regrid."""
    T = cfg.T if T is None else T
    n = tuple(cfg.n)
    w, c, B = initial_density(cfg.prior_mean[b], cfg.prior_cov, n, cfg.k_sigma, grid)
    rec = {"mean": [], "cov": [], "logC": [], "c": [], "B": [], "w": []}
    for k in range(T + 1):
        if k > 0:
            w, c, B = predict(w, c, B, cfg.A, cfg.Q, cfg.tau, cfg.l, diff_mode, trace_sign, step)
        lik = make_likelihood(cfg, grid_points(c, B, n), zs[k, b])
        w, logC = update(w, c, B, lik)
        mean, cov = moments(w, c, B)
        rec["mean"].append(mean)
        rec["cov"].append(cov)
        rec["logC"].append(logC)
        rec["c"].append(np.array(c))
        rec["B"].append(np.array(B))
        if keep_weights:
            rec["w"].append(w.copy())
        c2, B2 = regrid_target(mean, cov, n, cfg.k_sigma, grid)
        w = regrid(w, c, B, c2, B2)
        c, B = c2, B2
    rec["final"] = (w, c, B)
    return rec

"""Pins of the oracle's eigen-aligned grid design (R28: the
covariance-eigenvector grids of the refs of P:346) against what the definition fixes
independently of the eigensolver: the scaled grid matrix squares to the covariance,
its columns are orthogonal, a diagonal covariance gives R12's axis-aligned grid, and a
known rotation gives known columns (axis assignment and sign convention)."""
import math

import numpy as np
import pytest

from oracle import pmf_oracle as O


def _rot(theta):
    c, s = math.cos(theta), math.sin(theta)
    return np.array([[c, -s], [s, c]])


@pytest.mark.parametrize("nx", [1, 2, 3, 4])
def test_diagonal_cov_gives_axis_grid(nx):
    rng = np.random.default_rng(nx)
    cov = np.diag(rng.uniform(0.2, 3.0, nx))
    n = (32, 64, 16, 48)[:nx]
    c1, B1 = O.eigen_grid(np.zeros(nx), cov, n, 6.0)
    c2, B2 = O.design_grid(np.zeros(nx), cov, n, 6.0)
    assert np.allclose(B1, B2, rtol=1e-15, atol=0.0)


@pytest.mark.parametrize("nx", [2, 3, 4])
def test_scaled_grid_squares_to_cov(nx):
    """B diag(N) (B diag(N))^T = (2 k_sigma)^2 cov, columns orthogonal, det > 0 per column sign."""
    rng = np.random.default_rng(10 + nx)
    G = rng.standard_normal((nx, nx))
    cov = G @ G.T + 0.3 * np.eye(nx)
    n = np.array((32, 64, 16, 48)[:nx])
    ks = 6.0
    _, B = O.eigen_grid(np.zeros(nx), cov, tuple(n), ks)
    Bs = B * n[None, :]
    assert np.allclose(Bs @ Bs.T, 4 * ks * ks * cov, rtol=1e-13, atol=1e-13 * np.max(cov))
    gram = Bs.T @ Bs
    assert np.allclose(gram - np.diag(np.diag(gram)), 0.0, atol=1e-12 * np.max(gram))
    # each column's largest-magnitude component is positive and on a distinct axis
    axes = [int(np.argmax(np.abs(B[:, a]))) for a in range(nx)]
    assert all(B[axes[a], a] > 0 for a in range(nx))


@pytest.mark.parametrize("theta", [0.3, -0.5, 1.2])
def test_known_rotation(theta):
    """cov = R diag(9, 1) R^T: the major axis (cos, sin) goes to the axis it is nearest
    to, the minor axis to the other, both signed positive on their own axis."""
    cov = _rot(theta) @ np.diag([9.0, 1.0]) @ _rot(theta).T
    n = (64, 32)
    ks = 5.0
    _, B = O.eigen_grid(np.array([1.0, -2.0]), cov, n, ks)
    major = np.array([math.cos(theta), math.sin(theta)])
    minor = np.array([-math.sin(theta), math.cos(theta)])
    if abs(major[0]) >= abs(major[1]):
        a_major, a_minor = 0, 1
    else:
        a_major, a_minor = 1, 0
    major *= np.sign(major[a_major])
    minor *= np.sign(minor[a_minor])
    assert np.allclose(B[:, a_major], major * 2 * ks * 3.0 / n[a_major], rtol=1e-14, atol=1e-15)
    assert np.allclose(B[:, a_minor], minor * 2 * ks * 1.0 / n[a_minor], rtol=1e-14, atol=1e-15)


def test_conjugate_update_on_eigen_grid_matches_kalman():
    """P8 on the eigen-aligned grid of a correlated prior: Gaussian prior x linear-Gaussian
    likelihood -> the Kalman posterior mean, covariance and normaliser."""
    m0 = np.array([0.5, -1.0])
    P0 = np.array([[2.0, 1.2], [1.2, 1.0]])
    H = np.array([[1.0, 0.3]])
    R = np.array([[0.4]])
    z = np.array([0.9])
    n = (128, 128)
    w, c, B = O.initial_density(m0, P0, n, 8.0, O.GRID_EIGEN)
    assert abs(B[0, 1]) > 0.1 * abs(B[0, 0])           # the grid is really rotated
    lik = O.lik_linear_gauss(O.grid_points(c, B, n), z, H, R)
    w2, logC = O.update(w, c, B, lik)
    mean, cov = O.moments(w2, c, B)
    S = H @ P0 @ H.T + R
    K = P0 @ H.T @ np.linalg.inv(S)
    mk = m0 + (K @ (z - H @ m0))
    Pk = P0 - K @ H @ P0
    logN = -0.5 * (math.log(2 * math.pi * S[0, 0]) + float((z - H @ m0) @ np.linalg.solve(S, z - H @ m0)))
    assert np.allclose(mean, mk, atol=1e-12)
    assert np.allclose(cov, Pk, atol=1e-12)
    assert abs(logC - logN) < 1e-12

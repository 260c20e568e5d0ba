"""GPU parity of the eigen-aligned grid policy (pmf_config.grid = PMF_GRID_EIGEN, R28,
SURVEY 8(f) NEXT-4) against the oracle's eigen_grid on the same seeded inputs, on
every path: resident (2-D 128^2 batch), pencil (2-D), plane (3-D, 4-D). The grids
rotate with the posterior covariance, so every regrid is a general (non-separable)
map and every predict has cross terms. Priors are correlated with distinct
eigenvalues (a degenerate eigenspace has no unique aligned basis; DESIGN R28)."""
import numpy as np
import pytest

from oracle import pmf_oracle as O
from paper_2412_07240_b200 import pmf
from workloads import make_config, simulate

from parity_util import TOL, compare_runs, run_gpu

pytestmark = pytest.mark.gpu

P2 = np.array([[1.0, 0.3], [0.3, 0.25]])
P3 = np.array([[0.30, 0.05, 0.02], [0.05, 0.22, -0.03], [0.02, -0.03, 0.15]])
P4 = np.array([[1.0, 0.3, 0.1, 0.0], [0.3, 0.25, 0.0, 0.02], [0.1, 0.0, 0.6, 0.15], [0.0, 0.02, 0.15, 0.12]])


def _oracle(cfg, zs, T):
    return {b: O.run_filter(cfg, zs, b=b, T=T, keep_weights=True, grid=O.GRID_EIGEN) for b in range(cfg.batch)}


def _check(cfg, T, path, dtype="f64", tol=None):
    zs = simulate(cfg, T=T)["z"]
    g = run_gpu(cfg, zs, T, dtype=dtype, path=path, grid=pmf.GRID_EIGEN)
    assert g["filter"].path == path
    orc = _oracle(cfg, zs, T)
    # the grid really rotates
    assert max(abs(o["B"][k][1, 0]) for o in orc.values() for k in range(T + 1)) > 1e-3
    e = compare_runs(cfg, g, orc, T, TOL[dtype])
    t = TOL[dtype] if tol is None else tol
    assert e["w"] <= t and e["mean"] <= t and e["cov"] <= t and e["grid"] <= t, e
    if dtype == "f64":
        assert e["logC"] <= t, e


def test_eigen_grid_resident():
    cfg = make_config("C5", batch=4, prior_cov=P2)
    _check(cfg, 3, pmf.PATH_RESIDENT)


def test_eigen_grid_resident_f32():
    cfg = make_config("C5", batch=2, prior_cov=P2)
    _check(cfg, 2, pmf.PATH_RESIDENT, dtype="f32")


def test_eigen_grid_pencil():
    cfg = make_config("C2", n=(64, 64), prior_cov=P2)
    _check(cfg, 3, pmf.PATH_PENCIL)


def test_eigen_grid_plane_3d():
    cfg = make_config("C3", n=(32, 32, 16), prior_cov=P3)
    _check(cfg, 2, pmf.PATH_PLANE)


def test_eigen_grid_plane_4d():
    cfg = make_config("C4", n=(32, 32, 16, 16), prior_cov=P4)
    _check(cfg, 2, pmf.PATH_PLANE)


def test_eigen_grid_pencil_4d():
    cfg = make_config("C4", n=(16, 16, 16, 16), prior_cov=P4)
    _check(cfg, 2, pmf.PATH_PENCIL)


@pytest.mark.parametrize("cid, n, path, P", [("C5", (128, 128), pmf.PATH_RESIDENT, P2),
                                             ("C4", (32, 32, 16, 16), pmf.PATH_PLANE, P4),
                                             ("C1", (64,), pmf.PATH_AUTO, np.array([[0.3]]))])
def test_eigen_grid_with_crank_nicolson(cid, n, path, P):
    """R28 combined with Crank-Nicolson substeps (R27): both options at once, every path
    that takes them (nx = 1 runs the single-kernel epoch)."""
    over = {"n": n, "prior_cov": P}
    if cid == "C5":
        over["batch"] = 2
    cfg = make_config(cid, **over)
    T = 2
    zs = simulate(cfg, T=T)["z"]
    g = run_gpu(cfg, zs, T, path=path, grid=pmf.GRID_EIGEN, step=pmf.STEP_CN)
    orc = {b: O.run_filter(cfg, zs, b=b, T=T, keep_weights=True, grid=O.GRID_EIGEN, step=O.STEP_CN)
           for b in range(cfg.batch)}
    e = compare_runs(cfg, g, orc, T, TOL["f64"])
    assert max(e.values()) <= 1e-10, e

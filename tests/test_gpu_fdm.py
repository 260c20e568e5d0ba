"""GPU parity of the FDM baseline predictor (PMF_DIFF_FDM: eq:FST P:199-202 with
DST-I on FP64 tensor cores) against the CPU oracle's DIFF_FDM mode on the same
seeded inputs, through the C ABI. Bar as elsewhere: relative L-inf of the weights
normalised by the peak <= 1e-10 (fp64); moments, log-normaliser, grid likewise."""
import numpy as np
import pytest

from oracle import pmf_oracle as O
from paper_2412_07240_b200 import pmf
from workloads import make_config, random_density, simulate

from parity_util import compare_runs, run_gpu

pytestmark = pytest.mark.gpu

# The explicit scheme is stable only for a_m = Q_mm dt / (2 delta_m^2) <= 1/4 (CFL).
# C1's posterior grid (delta ~ 0.1) needs dt <= 0.005: its FDM case uses N = 32 and
# l = 64 substeps per interval (a ~ 0.08); with l = 10 the FDM density blows up.
CASES = {
    "C1_32_l64": ("C1", {"n": (32,), "l": 64}, 5),
    "C5_b3_32x64": ("C5", {"batch": 3, "n": (32, 64)}, 3),
    "C3_32x32x32": ("C3", {"n": (32, 32, 32)}, 2),
    "C4_32x32x32x32": ("C4", {"n": (32, 32, 32, 32)}, 1),
    "C4_96x32x32x64": ("C4", {"n": (96, 32, 32, 64)}, 1),
    "C2_128x96": ("C2", {"n": (128, 96)}, 2),
}


@pytest.mark.parametrize("name", list(CASES))
def test_fdm_filter_run_parity(name):
    cid, over, T = CASES[name]
    cfg = make_config(cid, **over)
    zs = simulate(cfg, T=T)["z"]
    g = run_gpu(cfg, zs, T, diff_mode=pmf.DIFF_FDM)
    orc = {b: O.run_filter(cfg, zs, b=b, T=T, keep_weights=True, diff_mode=O.DIFF_FDM)
           for b in range(cfg.batch)}
    e = compare_runs(cfg, g, orc, T, 1e-10)
    assert e["w"] <= 1e-10, e
    assert e["mean"] <= 1e-10 and e["cov"] <= 1e-10 and e["logC"] <= 1e-10 and e["grid"] <= 1e-10, e


@pytest.mark.parametrize("nx,n", [(1, (96,)), (2, (64, 32)), (3, (32, 64, 32))])
def test_fdm_predict_operator_sheared(nx, n):
    """One FDM predict from a non-Gaussian density on a sheared grid with non-zero A
    (moving grid: the axis spacings change every substep, the eigenvectors do not);
    stable step (a_m <= 0.15)."""
    rng = np.random.default_rng(70 + nx)
    A = 0.5 * rng.standard_normal((nx, nx))
    Q = np.diag(rng.uniform(0.01, 0.05, nx))
    B = np.diag(rng.uniform(0.05, 0.1, nx)) + 0.01 * rng.standard_normal((nx, nx))
    c = rng.standard_normal(nx)
    wlib = random_density(n, 1, seed=5)[0]
    f = pmf.Filter(nx, n, A, Q, diff_mode=pmf.DIFF_FDM)
    f.set_state(c[None], B[None], wlib)
    tau, l = 0.3, 20
    f.predict(tau / l, l)
    w_gpu = f.weights()[0]
    cg, Bg = f.grid()
    w_log = O.from_lib(wlib, n)
    wo, co, Bo = O.predict(w_log, c, B, A, Q, tau, l, diff_mode=O.DIFF_FDM)
    wo = O.to_lib(wo)
    assert float(np.max(np.abs(w_gpu - wo)) / np.max(np.abs(wo))) <= 1e-12
    assert np.max(np.abs(cg[0] - co)) <= 1e-13 and np.max(np.abs(Bg[0] - Bo)) <= 1e-13


def test_fdm_rejects_unsupported():
    cfg = make_config("C2")       # 256^2: not a DST size the FDM kernels hold
    with pytest.raises(pmf.PMFError):
        pmf.Filter(cfg.nx, cfg.n, cfg.A, cfg.Q, diff_mode=pmf.DIFF_FDM)
    cfg = make_config("C5", batch=2)
    with pytest.raises(pmf.PMFError):
        pmf.Filter(cfg.nx, cfg.n, cfg.A, cfg.Q, batch=2, dtype="f32", diff_mode=pmf.DIFF_FDM)
    Qnd = np.array([[0.1, 0.02], [0.02, 0.1]])
    with pytest.raises(pmf.PMFError):
        pmf.Filter(2, (32, 32), cfg.A, Qnd, diff_mode=pmf.DIFF_FDM)

"""GPU parity of the plane path (PMF_PATH_PLANE: (i0,i1)-plane kernels, strided
passes, regrid fused into the forward pass) against the CPU oracle on the same
seeded inputs, through the C ABI. Bar: relative L-inf of the weights normalised
by the peak density <= 1e-10 (fp64) / 1e-4 (fp32); same bounds for mean (per
sqrt of the largest eigenvalue), covariance, log-normaliser and grid.

Shapes span the register-FFT sizes (plane 32/64/96/128, strided axes 16..128),
the row-separable regrid (CV models: C4) and the general gather (dense A: C3)."""
import numpy as np
import pytest

from paper_2412_07240_b200 import pmf
from workloads import make_config, simulate

from parity_util import TOL, compare_runs, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

CASES = {
    # name: (config id, overrides, T)
    "C3_32x32x16": ("C3", {"n": (32, 32, 16)}, 3),
    "C3_64x64x32": ("C3", {"n": (64, 64, 32)}, 2),
    "C3_128x128x16": ("C3", {"n": (128, 128, 16)}, 2),
    "C3_96x96x64": ("C3", {"n": (96, 96, 64)}, 1),
    "C4_32x32x16x16": ("C4", {"n": (32, 32, 16, 16)}, 3),
    "C4_96x96x16x32": ("C4", {"n": (96, 96, 16, 32)}, 1),
    "C4_64x64x32x16": ("C4", {"n": (64, 64, 32, 16)}, 2),
    "C4_b2_32": ("C4", {"n": (32, 32, 16, 16), "batch": 2}, 2),
    # n2 = n3, fp64: the three-pass transposed-spectrum route (kernels_quad.cu)
    "C4_32x32x32x32": ("C4", {"n": (32, 32, 32, 32)}, 2),
    "C4_32x32x64x64": ("C4", {"n": (32, 32, 64, 64)}, 1),
    "C4_32x32x96x96": ("C4", {"n": (32, 32, 96, 96)}, 1),
    "C4_64x64x16x16": ("C4", {"n": (64, 64, 16, 16)}, 2),
    "C4_64x64x32x32": ("C4", {"n": (64, 64, 32, 32)}, 1),
    "C4_96x96x16x16": ("C4", {"n": (96, 96, 16, 16)}, 2),
    "C4_b3_96x96x32x32": ("C4", {"n": (96, 96, 32, 32), "batch": 3}, 1),
}


QUAD = ("C4_32x32x16x16", "C4_b2_32", "C4_32x32x32x32", "C4_96x96x16x16", "C4_b3_96x96x32x32")


@pytest.fixture
def five_pass(monkeypatch):
    """Force the per-plane-layout five-pass route (read by the library on every call)."""
    monkeypatch.setenv("PMF_NO_QUAD", "1")


@pytest.mark.parametrize("name", list(CASES))
def test_plane_run_parity_f64(name):
    cid, over, T = CASES[name]
    cfg = make_config(cid, **over)
    zs = simulate(cfg, T=T)["z"]
    g = run_gpu(cfg, zs, T, path=pmf.PATH_PLANE)
    assert g["filter"].path == pmf.PATH_PLANE
    orc = run_oracle(cfg, zs, T)
    e = compare_runs(cfg, g, orc, T, TOL["f64"])
    assert e["w"] <= 1e-10, e
    assert e["mean"] <= 1e-10 and e["cov"] <= 1e-10 and e["logC"] <= 1e-10 and e["grid"] <= 1e-10, e


@pytest.mark.parametrize("name", QUAD)
def test_plane_five_pass_parity_f64(name, five_pass):
    """The per-plane-layout five-pass route (the fallback for shapes the three-pass route
    does not take) on the three-pass route's shapes: same bar against the oracle."""
    test_plane_run_parity_f64(name)


@pytest.mark.parametrize("name", ["C4_32x32x16x16", "C4_96x96x16x16"])
def test_plane_three_vs_five_pass(name, monkeypatch):
    """The two nx = 4 routes agree to rounding (1e-12) on weights, moments and normaliser."""
    cid, over, T = CASES[name]
    cfg = make_config(cid, **over)
    zs = simulate(cfg, T=T)["z"]
    a = run_gpu(cfg, zs, T, path=pmf.PATH_PLANE)
    monkeypatch.setenv("PMF_NO_QUAD", "1")
    b = run_gpu(cfg, zs, T, path=pmf.PATH_PLANE)
    wa, wb = a["filter"].weights(), b["filter"].weights()
    assert float(np.max(np.abs(wa - wb)) / np.max(np.abs(wb))) < 1e-12
    for k in range(T + 1):
        assert np.max(np.abs(a["mean"][k] - b["mean"][k])) < 1e-12
        assert abs(float(a["logC"][k][0]) - float(b["logC"][k][0])) < 1e-12


@pytest.mark.parametrize("name", ["C3_32x32x16", "C4_32x32x16x16", "C4_32x32x32x32"])
def test_plane_run_parity_f32(name):
    cid, over, T = CASES[name]
    cfg = make_config(cid, **over)
    zs = simulate(cfg, T=T)["z"]
    g = run_gpu(cfg, zs, T, dtype="f32", path=pmf.PATH_PLANE)
    orc = run_oracle(cfg, zs, T)
    e = compare_runs(cfg, g, orc, T, TOL["f32"])
    assert e["w"] <= 1e-4 and e["mean"] <= 1e-4 and e["cov"] <= 1e-4, e


@pytest.mark.parametrize("cid", ["C3", "C4"])
def test_plane_full_size_matches_pencil(cid):
    """BASELINE sizes (128^3, 96^4): the plane path agrees with the pencil path
    (itself parity-tested against the oracle) on every epoch's moments and
    normaliser, and on the final weights element by element."""
    cfg = make_config(cid)
    T = 2
    zs = simulate(cfg, T=T)["z"]
    a = run_gpu(cfg, zs, T, path=pmf.PATH_PLANE, keep_weights=False)
    b = run_gpu(cfg, zs, T, path=pmf.PATH_PENCIL, keep_weights=False)
    for k in range(T + 1):
        sd = np.sqrt(np.max(np.linalg.eigvalsh(b["cov"][k][0])))
        assert np.max(np.abs(a["mean"][k] - b["mean"][k])) / sd < 1e-11
        assert np.max(np.abs(a["cov"][k] - b["cov"][k])) / np.max(np.abs(b["cov"][k])) < 1e-11
        assert abs(float(a["logC"][k][0]) - float(b["logC"][k][0])) < 1e-11
    wa, wb = a["filter"].weights(), b["filter"].weights()
    assert float(np.max(np.abs(wa - wb)) / np.max(np.abs(wb))) < 1e-11


def test_plane_predict_only_normalisation():
    """predict without an update: the closed-form normalisation (Alg. 6) gives a
    density that integrates to one and equals the pencil path's."""
    cfg = make_config("C4", n=(32, 32, 16, 16))
    outs = []
    for path in (pmf.PATH_PLANE, pmf.PATH_PENCIL):
        f = pmf.Filter(cfg.nx, cfg.n, cfg.A, cfg.Q, path=path)
        f.set_gaussian(cfg.prior_mean, cfg.prior_cov[None], cfg.k_sigma)
        f.predict(cfg.tau / cfg.l, cfg.l)
        outs.append(f.weights()[0])
        c, B = f.grid()
        vol = abs(np.linalg.det(B[0]))
        assert abs(vol * outs[-1].sum() - 1.0) < 1e-12
    assert float(np.max(np.abs(outs[0] - outs[1])) / np.max(np.abs(outs[1]))) < 1e-12

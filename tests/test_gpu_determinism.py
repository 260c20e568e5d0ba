"""Run-to-run determinism of every kernel family: the same seeded run three times from
fresh contexts must give bitwise-equal weights, moments and normalisers. Every reduction
in the library has a fixed order (per-block partials summed in index order, the virtual
all-reduce in rank order), so any difference is a data race -- between the threads of a
kernel, or between the compute stream and the exchange stream of the pipelined sharded
route. (compute-sanitizer's racecheck is not available on the GPU pool; this is the
check that stands in for it, at sizes that fill the device: several CTA rounds, several
exchange chunks in flight.)"""
import numpy as np
import pytest

from paper_2412_07240_b200 import pmf
from workloads import make_config, simulate

from parity_util import run_gpu

pytestmark = pytest.mark.gpu

# name: (config, overrides, T, dtype, path, filter kwargs, expected kernel family)
CASES = {
    "line": ("C1", {}, 6, "f64", pmf.PATH_AUTO, {}, "line"),
    "cluster": ("C2", {}, 3, "f64", pmf.PATH_AUTO, {}, "cluster"),
    "resident_3_rounds": ("C5", {"batch": 300}, 3, "f64", pmf.PATH_AUTO, {}, "resident"),
    "resident_f32": ("C5", {"batch": 300}, 3, "f32", pmf.PATH_AUTO, {}, "resident"),
    "resident_cn": ("C5", {"batch": 160}, 2, "f64", pmf.PATH_AUTO, {"step": pmf.STEP_CN}, "resident"),
    "plane3": ("C3", {"n": (64, 64, 32)}, 3, "f64", pmf.PATH_PLANE, {}, "plane"),
    "plane4_five_pass": ("C4", {"n": (64, 64, 32, 16)}, 2, "f64", pmf.PATH_PLANE, {}, "plane"),
    "quad_three_pass": ("C4", {"n": (32, 32, 32, 32)}, 3, "f64", pmf.PATH_PLANE, {}, "plane"),
    "quad_96": ("C4", {"n": (96, 96, 16, 16)}, 2, "f64", pmf.PATH_PLANE, {}, "plane"),
    "pencil17_terrain": ("C6", {"n": (34, 18, 34, 18)}, 3, "f64", pmf.PATH_AUTO, {}, "pencil"),
    "fdm": ("C5", {"batch": 9}, 2, "f64", pmf.PATH_AUTO, {"diff_mode": pmf.DIFF_FDM}, "fdm"),
    "sharded_quad_x4": ("C4", {"n": (32, 32, 32, 32)}, 3, "f64", pmf.PATH_PENCIL,
                        {"world": 4, "sharded": True}, "sharded"),
    "sharded_quad96_x8": ("C4", {"n": (96, 96, 16, 16)}, 2, "f64", pmf.PATH_PENCIL,
                          {"world": 8, "sharded": True}, "sharded"),
    "sharded_pencil_x2": ("C3", {"n": (16, 12, 24)}, 3, "f64", pmf.PATH_PENCIL,
                          {"world": 2, "sharded": True}, "sharded"),
}


@pytest.mark.parametrize("name", list(CASES))
def test_three_runs_bitwise_equal(name):
    cid, over, T, dtype, path, kw, family = CASES[name]
    cfg = make_config(cid, **over)
    zs = simulate(cfg, T=T)["z"]
    runs = []
    for _ in range(3):
        g = run_gpu(cfg, zs, T, dtype=dtype, path=path, **kw)
        assert g["filter"].epoch_kernel == family, g["filter"].epoch_kernel
        g["filter"].close()
        runs.append(g)
    a = runs[0]
    assert all(np.isfinite(w).all() for w in a["w"])
    for b in runs[1:]:
        for k in range(T + 1):
            assert np.array_equal(a["w"][k], b["w"][k]), (name, k)
            assert np.array_equal(a["mean"][k], b["mean"][k]) and np.array_equal(a["cov"][k], b["cov"][k]), (name, k)
            assert np.array_equal(a["logC"][k], b["logC"][k]), (name, k)
            assert np.array_equal(a["c"][k], b["c"][k]) and np.array_equal(a["B"][k], b["B"][k]), (name, k)


@pytest.mark.parametrize("kw", [{}, {"world": 4, "sharded": True}], ids=["plane", "sharded_x4"])
def test_full_size_c4_moments_bitwise_equal(kw):
    """The bench configuration itself (96^4, every SM busy, 4 exchange chunks in flight on
    the sharded route): moments, normaliser and grid of 3 epochs, two runs, bitwise."""
    cfg = make_config("C4")
    T = 2
    zs = simulate(cfg, T=T)["z"]
    runs = []
    for _ in range(2):
        g = run_gpu(cfg, zs, T, path=pmf.PATH_PENCIL if kw else pmf.PATH_AUTO, keep_weights=False, **kw)
        g["filter"].close()
        runs.append(g)
    a, b = runs
    for k in range(T + 1):
        assert np.isfinite(a["mean"][k]).all() and np.isfinite(a["logC"][k]).all()
        for key in ("mean", "cov", "logC", "c", "B"):
            assert np.array_equal(a[key][k], b[key][k]), (key, k)

"""GPU parity: the CUDA path through the C ABI vs the CPU oracle on the same
seeded inputs (element-wise weights, moments, normaliser, grid) -- bar: relative
L-inf normalised by the peak density <= 1e-10 (fp64), <= 1e-4 (fp32)."""
import numpy as np
import pytest

from oracle import pmf_oracle as O
from paper_2412_07240_b200 import pmf
from workloads import make_config, random_density, simulate

from parity_util import TOL, compare_runs, lik_of, make_filter, rel_linf, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

CASES = {
    # name: (config id, overrides, T)   sizes span several tiles + ragged tails, radix 2 and 3
    "C1": ("C1", {}, 20),
    "C1b3": ("C1", {"batch": 3, "n": (96,)}, 5),
    "C2s": ("C2", {"n": (48, 32)}, 6),
    "C3s": ("C3", {"n": (16, 12, 24)}, 4),
    "C4s": ("C4", {"n": (8, 6, 12, 8)}, 3),
    "C5s": ("C5", {"batch": 5, "n": (24, 32)}, 4),
    # the paper's own grid sizes (N_pa = 34; N = 80, 200 in Figs. 2-3):
    # radix 17, 5 and 5^2 stages, and 7, 11, 13
    "C1_34": ("C1", {"n": (34,)}, 5),
    "C1_80": ("C1", {"n": (80,)}, 4),
    "C1_200": ("C1", {"n": (200,)}, 3),
    "C5_34x28": ("C5", {"batch": 2, "n": (34, 28)}, 3),
    "C3_22x26x14": ("C3", {"n": (22, 26, 14)}, 2),
    "C4_34x10x34x10": ("C4", {"n": (34, 10, 34, 10)}, 2),
    # the paper's §VI scenario (NEXT-3): coordinated turn, terrain-map altitude with
    # Gaussian-mixture noise, N_pa = 34 (full size) and a thinner variant
    "C6_34x18x34x18": ("C6", {"n": (34, 18, 34, 18)}, 3),
    "C6": ("C6", {}, 1),
}


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("path", [pmf.PATH_PENCIL, pmf.PATH_AUTO])
def test_filter_run_parity_f64(name, path):
    cid, over, T = CASES[name]
    cfg = make_config(cid, **over)
    zs = simulate(cfg, T=T)["z"]
    g = run_gpu(cfg, zs, T, path=path)
    orc = run_oracle(cfg, zs, T)
    e = compare_runs(cfg, g, orc, T, TOL["f64"])
    assert e["w"] <= 1e-10, e
    assert e["mean"] <= 1e-10 and e["cov"] <= 1e-10 and e["logC"] <= 1e-10 and e["grid"] <= 1e-10, e


@pytest.mark.parametrize("name", ["C2s", "C5s"])
def test_filter_run_parity_f32(name):
    cid, over, T = CASES[name]
    cfg = make_config(cid, **over)
    zs = simulate(cfg, T=T)["z"]
    g = run_gpu(cfg, zs, T, dtype="f32")
    orc = run_oracle(cfg, zs, T)
    e = compare_runs(cfg, g, orc, T, TOL["f32"])
    assert e["w"] <= 1e-4 and e["mean"] <= 1e-4 and e["cov"] <= 1e-4, e


def test_step_api_equals_unfused_sequence():
    cfg = make_config("C5", batch=3, n=(24, 32))
    T = 3
    zs = simulate(cfg, T=T)["z"]
    a = run_gpu(cfg, zs, T)
    b = run_gpu(cfg, zs, T, use_step=True)
    for k in range(T + 1):
        assert np.max(np.abs(a["mean"][k] - b["mean"][k])) < 1e-12
        assert np.max(np.abs(a["logC"][k] - b["logC"][k])) < 1e-12


@pytest.mark.parametrize("nx,n", [(2, (32, 24)), (3, (12, 16, 8))])
@pytest.mark.parametrize("mode", ["full", "axis_literal", "printed_trace"])
def test_predict_operator_parity_sheared(nx, n, mode):
    """One predict from a non-Gaussian density on a sheared grid with
    non-diagonal A (and Q for the full mode)."""
    rng = np.random.default_rng(11 + nx)
    A = 0.5 * rng.standard_normal((nx, nx))
    if mode == "axis_literal":
        Q = np.diag(rng.uniform(0.05, 0.3, nx))
    else:
        M = rng.standard_normal((nx, nx))
        Q = 0.05 * (M @ M.T) + 0.02 * np.eye(nx)
    B = np.diag(rng.uniform(0.05, 0.1, nx)) + 0.01 * rng.standard_normal((nx, nx))
    c = rng.standard_normal(nx)
    wlib = random_density(n, 1, seed=3)[0]
    diff = O.DIFF_AXIS_LITERAL if mode == "axis_literal" else O.DIFF_FULL
    ts = O.TRACE_SIGN_PRINTED if mode == "printed_trace" else O.TRACE_SIGN_PHYSICAL
    f = pmf.Filter(nx, n, A, Q, diff_mode=diff, trace_sign=ts)
    f.set_state(c[None], B[None], wlib)
    tau, l = 0.3, 7
    f.predict(tau / l, l)
    wg = f.weights()[0]
    cg, Bg = f.grid()
    w0 = O.normalise(O.from_lib(wlib, n), B)
    wo, co, Bo = O.predict(w0, c, B, A, Q, tau, l, diff_mode=diff, trace_sign=ts)
    assert rel_linf(wg, O.to_lib(wo)) <= 1e-10
    assert rel_linf(Bg[0], Bo) <= 1e-13 and rel_linf(cg[0], co) <= 1e-13


def test_update_and_regrid_operator_parity():
    """Standalone update (range likelihood) and regrid on a sheared grid."""
    n = (18, 16, 12)
    cfg = make_config("C3", n=n)
    rng = np.random.default_rng(5)
    B = np.diag([0.12, 0.1, 0.11]) + 0.02 * rng.standard_normal((3, 3))
    c = np.array([1.5, 0.2, -0.1])
    wlib = random_density(n, 1, seed=9)[0]
    f = pmf.Filter(3, n, cfg.A, cfg.Q)
    f.set_state(c[None], B[None], wlib)
    z = np.array([[1.6]])
    f.update(z, lik_of(cfg))
    mean, cov, logc = f.moments()
    w0 = O.normalise(O.from_lib(wlib, n), B)
    X = O.grid_points(c, B, n)
    wo, lo = O.update(w0, c, B, O.lik_range_gauss(X, z[0], cfg.sigma))
    mo, co = O.moments(wo, c, B)
    assert rel_linf(f.weights()[0], O.to_lib(wo)) <= 1e-10
    assert abs(logc[0] - lo) <= 1e-10 and rel_linf(mean[0], mo) <= 1e-10 and rel_linf(cov[0], co) <= 1e-10
    f.regrid(4.0)
    wg = f.weights()[0]
    cg, Bg = f.grid()
    c2, B2 = O.regrid_target(mo, co, n, 4.0)
    wr = O.regrid(wo, c, B, c2, B2)
    assert rel_linf(wg, O.to_lib(wr)) <= 1e-10
    assert rel_linf(Bg[0], B2) <= 1e-12


def test_error_codes():
    cfg = make_config("C1")
    f = pmf.Filter(1, cfg.n, cfg.A, cfg.Q)
    with pytest.raises(pmf.PMFError) as e:
        f.predict(0.01, 10)
    assert e.value.code == -8                        # PMF_E_STATE
    f.set_gaussian(cfg.prior_mean, cfg.prior_cov[None], cfg.k_sigma)
    with pytest.raises(pmf.PMFError) as e:
        f.predict(-1.0, 10)
    assert e.value.code == -7                        # PMF_E_DT
    with pytest.raises(pmf.PMFError) as e:
        f.regrid(6.0)
    assert e.value.code == -8
    f.update(np.array([[1e6]]), lik_of(cfg))          # far outside the support: normaliser underflows to 0
    with pytest.raises(pmf.PMFError) as e:
        f.moments()
    assert e.value.code == -6                        # PMF_E_NO_SUPPORT


def test_launch_count_and_determinism():
    cfg = make_config("C5", batch=4, n=(32, 32))
    zs = simulate(cfg, T=2)["z"]
    a = run_gpu(cfg, zs, 2)
    b = run_gpu(cfg, zs, 2)
    assert a["filter"].launches > 0
    for k in range(3):
        assert np.array_equal(a["w"][k], b["w"][k])          # fixed-order reductions: bitwise
        assert np.array_equal(a["mean"][k], b["mean"][k])


# ----------------------------------------------------------------------------- resident (fused) path
@pytest.mark.parametrize("use_step", [False, True])
def test_resident_epoch_parity_f64(use_step):
    """The one-launch-per-epoch kernel (regrid + predict + update + moments) on
    128x128 filters, batch not a multiple of anything, vs the oracle."""
    cfg = make_config("C5", batch=7)
    T = 3
    zs = simulate(cfg, T=T)["z"]
    g = run_gpu(cfg, zs, T, path=pmf.PATH_RESIDENT, use_step=use_step)
    assert g["filter"].path == pmf.PATH_RESIDENT
    orc = run_oracle(cfg, zs, T)
    e = compare_runs(cfg, g, orc, T, TOL["f64"])
    assert e["w"] <= 1e-10 and e["mean"] <= 1e-10 and e["cov"] <= 1e-10 and e["logC"] <= 1e-10, e
    assert e["grid"] <= 1e-10, e


def test_resident_epoch_parity_f32():
    cfg = make_config("C5", batch=5)
    T = 3
    zs = simulate(cfg, T=T)["z"]
    g = run_gpu(cfg, zs, T, dtype="f32", path=pmf.PATH_RESIDENT)
    orc = run_oracle(cfg, zs, T)
    e = compare_runs(cfg, g, orc, T, TOL["f32"])
    assert e["w"] <= 1e-4 and e["mean"] <= 1e-4 and e["cov"] <= 1e-4, e


@pytest.mark.parametrize("mode", ["full", "axis_literal", "printed_trace"])
def test_resident_predict_operator_parity_sheared(mode):
    """Predict only (no update) on a sheared 128x128 grid, non-diagonal A and Q,
    a non-Gaussian input: exercises the resident kernel's UPDATE=0 branch."""
    nx, n = 2, (128, 128)
    rng = np.random.default_rng(21)
    A = 0.5 * rng.standard_normal((nx, nx))
    if mode == "axis_literal":
        Q = np.diag(rng.uniform(0.05, 0.3, nx))
    else:
        M = rng.standard_normal((nx, nx))
        Q = 0.05 * (M @ M.T) + 0.02 * np.eye(nx)
    B = np.diag(rng.uniform(0.02, 0.03, nx)) + 0.003 * rng.standard_normal((nx, nx))
    c = rng.standard_normal(nx)
    wlib = random_density(n, 2, seed=4)
    diff = O.DIFF_AXIS_LITERAL if mode == "axis_literal" else O.DIFF_FULL
    ts = O.TRACE_SIGN_PRINTED if mode == "printed_trace" else O.TRACE_SIGN_PHYSICAL
    f = pmf.Filter(nx, n, A, Q, batch=2, diff_mode=diff, trace_sign=ts, path=pmf.PATH_RESIDENT)
    f.set_state(np.stack([c, -c]), np.stack([B, B.T]), wlib)
    tau, l = 0.3, 7
    f.predict(tau / l, l)
    wg = f.weights()
    cg, Bg = f.grid()
    for b, (cb, Bb) in enumerate([(c, B), (-c, B.T)]):
        w0 = O.normalise(O.from_lib(wlib[b], n), Bb)
        wo, co, Bo = O.predict(w0, cb, Bb, A, Q, tau, l, diff_mode=diff, trace_sign=ts)
        assert rel_linf(wg[b], O.to_lib(wo)) <= 1e-10
        assert rel_linf(Bg[b], Bo) <= 1e-13 and rel_linf(cg[b], co) <= 1e-13


def test_resident_matches_pencil_path():
    cfg = make_config("C5", batch=3)
    T = 2
    zs = simulate(cfg, T=T)["z"]
    a = run_gpu(cfg, zs, T, path=pmf.PATH_RESIDENT)
    b = run_gpu(cfg, zs, T, path=pmf.PATH_PENCIL)
    for k in range(T + 1):
        assert rel_linf(a["w"][k], b["w"][k]) <= 1e-12


@pytest.mark.parametrize("cid,over", [("C1", {}), ("C2", {"n": (48, 32)}), ("C5", {"batch": 3, "n": (128, 128)}),
                                      ("C4", {"n": (32, 32, 16, 16)})])
def test_graph_replay_bitwise_equal(cid, over):
    """CUDA-graph replay of pmf_step epochs (non-default stream) == direct launches,
    bit for bit, and the same kernel count."""
    import torch
    cfg = make_config(cid, **over)
    T = 4
    zs = simulate(cfg, T=T)["z"]
    lik = lik_of(cfg)
    outs = []
    for graphs in (True, False):
        s = torch.cuda.Stream()
        f = pmf.Filter(cfg.nx, cfg.n, cfg.A, cfg.Q, batch=cfg.batch, stream=s.cuda_stream)
        f.use_graphs(graphs)
        f.set_gaussian(cfg.prior_mean, np.broadcast_to(cfg.prior_cov, (cfg.batch, cfg.nx, cfg.nx)), cfg.k_sigma)
        f.update(zs[0], lik)
        f.regrid(cfg.k_sigma)
        l0 = f.launches
        for k in range(1, T + 1):
            f.step(cfg.tau / cfg.l, cfg.l, zs[k], lik, cfg.k_sigma)
        mean, cov, logc = f.moments()
        outs.append((f.weights(), mean, cov, logc, f.launches - l0))
        f.close()
    a, b = outs
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and np.array_equal(a[3], b[3])
    assert a[4] == b[4]


@pytest.mark.parametrize("cid,over", [("C5", {"batch": 3}), ("C4", {"n": (32, 32, 16, 16)}), ("C3", {"n": (16, 12, 24)})])
def test_graph_replay_varying_substeps(cid, over):
    """Graphs captured at l = 10 are not replayed after a predict with more substeps
    reallocated the substep table and coefficient buffers: l = 10 -> 100 -> 10
    with graphs on equals graphs off, bit for bit."""
    import torch
    cfg = make_config(cid, **over)
    T = 3
    zs = simulate(cfg, T=T)["z"]
    lik = lik_of(cfg)
    outs = []
    for graphs in (True, False):
        s = torch.cuda.Stream()
        f = pmf.Filter(cfg.nx, cfg.n, cfg.A, cfg.Q, batch=cfg.batch, stream=s.cuda_stream)
        f.use_graphs(graphs)
        f.set_gaussian(cfg.prior_mean, np.broadcast_to(cfg.prior_cov, (cfg.batch, cfg.nx, cfg.nx)), cfg.k_sigma)
        f.update(zs[0], lik)
        f.regrid(cfg.k_sigma)
        for k, l in zip(range(1, T + 1), (10, 100, 10)):
            f.step(cfg.tau / l, l, zs[k], lik, cfg.k_sigma)
        mean, cov, logc = f.moments()
        outs.append((f.weights(), mean, cov, logc))
        f.close()
    a, b = outs
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and np.array_equal(a[3], b[3])


@pytest.mark.parametrize("name", ["C1", "C2s", "C3s", "C4s", "C5s", "C3_plane_32", "C4_plane_32", "C5_resident",
                                  "C5_resident_step"])
def test_crank_nicolson_parity(name):
    """NEXT-4: Crank-Nicolson substeps (R27) through the C ABI vs the oracle's STEP_CN on
    the pencil, plane and resident kernels (the latter eager and through pmf_step)."""
    extra = {"C3_plane_32": ("C3", {"n": (32, 32, 16)}, 2), "C4_plane_32": ("C4", {"n": (32, 32, 16, 16)}, 2),
             "C5_resident": ("C5", {"batch": 3}, 3), "C5_resident_step": ("C5", {"batch": 3}, 3)}
    cid, over, T = extra.get(name) or CASES[name]
    cfg = make_config(cid, **over)
    zs = simulate(cfg, T=T)["z"]
    g = run_gpu(cfg, zs, T, step=pmf.STEP_CN, use_step=name.endswith("_step"))
    if name.startswith("C5_resident"):
        assert g["filter"].path == pmf.PATH_RESIDENT
    orc = {b: O.run_filter(cfg, zs, b=b, T=T, keep_weights=True, step=O.STEP_CN) for b in range(cfg.batch)}
    e = compare_runs(cfg, g, orc, T, 1e-10)
    assert e["w"] <= 1e-10, e
    assert e["mean"] <= 1e-10 and e["cov"] <= 1e-10 and e["logC"] <= 1e-10 and e["grid"] <= 1e-10, e


def _terrain_cfg_2d():
    """A 2-D variant of the §VI measurement (C6): state [px, py] with a CV-free drift,
    altitude from C6's synthetic map, Gaussian-mixture noise; resident-kernel size."""
    import dataclasses
    import workloads as W
    c6 = make_config("C6")
    cfg = make_config("C5", batch=2, n=(128, 128))
    return dataclasses.replace(cfg, A=np.array([[0.0, 0.0], [0.0, 0.0]]), Q=np.diag([4.0, 4.0]),
                               prior_mean=np.tile(c6.prior_mean[0, [0, 2]], (2, 1)),
                               prior_cov=np.diag([90.0, 60.0]), tau=1.0, lik_kind=W.LIK_TERRAIN_GM,
                               H=None, R=None, extra={"gm": c6.extra["gm"]}, seed=6)


def test_terrain_likelihood_resident_and_plane():
    """The terrain-GM likelihood (PMF_LIK_TERRAIN_GM) after the resident kernel (2-D,
    128^2) and after the plane kernels (C6 at 32x32x16x16), against the oracle."""
    import workloads as W
    orig_table = W.terrain_table
    c6 = make_config("C6")
    # 2-D: the C6 map with (ix, iy) = (0, 1)
    W.terrain_table = lambda cfg, **kw: orig_table(c6)[:5] + (0, 1)
    try:
        cfg = _terrain_cfg_2d()
        T = 2
        # static truth 3 m / 2 m off the prior mean: altitude + the mixture's two components
        px, py = cfg.prior_mean[0, 0] + 3.0, cfg.prior_mean[0, 1] - 2.0
        h = float(W.terrain_field(c6, px, py))
        zs = np.array([h + 0.3, h + 20.0 - 0.5, h - 0.2])[:, None, None] * np.ones((1, cfg.batch, 1))
        g = run_gpu(cfg, zs, T)
        assert g["filter"].path == pmf.PATH_RESIDENT
        orc = {b: O.run_filter(cfg, zs, b=b, T=T, keep_weights=True) for b in range(cfg.batch)}
        e = compare_runs(cfg, g, orc, T, 1e-10)
        assert e["w"] <= 1e-10 and e["mean"] <= 1e-10 and e["logC"] <= 1e-10, e
    finally:
        W.terrain_table = orig_table
    cfg = make_config("C6", n=(32, 32, 16, 16))
    T = 2
    zs = simulate(cfg, T=T)["z"]
    g = run_gpu(cfg, zs, T)
    assert g["filter"].path == pmf.PATH_PLANE
    orc = {0: O.run_filter(cfg, zs, b=0, T=T, keep_weights=True)}
    e = compare_runs(cfg, g, orc, T, 1e-10)
    assert e["w"] <= 1e-10 and e["mean"] <= 1e-10 and e["logC"] <= 1e-10, e


def test_moments_async_matches_moments():
    """pmf_moments_async: the same records as pmf_moments (mean, cov, log C, flag), read
    after a sync, with the pending regrid left pending (the next step still fuses it)."""
    import torch
    cfg = make_config("C5", batch=3)
    zs = simulate(cfg, T=2)["z"]
    f = make_filter(cfg)
    lik = lik_of(cfg)
    f.update(zs[0], lik)
    f.regrid(cfg.k_sigma)
    f.step(cfg.tau / cfg.l, cfg.l, zs[1], lik, cfg.k_sigma)
    n0 = f.launches
    buf = torch.empty(f.moments_bytes // 8, dtype=torch.float64).pin_memory()
    f.moments_async(buf)
    assert f.launches - n0 == 1          # the pack only: the recorded regrid stays pending
    torch.cuda.synchronize()
    mean, cov, logc = f.moments()
    rec = buf.numpy().reshape(cfg.batch, -1)
    nx = cfg.nx
    assert np.array_equal(rec[:, :nx], mean)
    assert np.array_equal(rec[:, nx:nx + nx * nx].reshape(cfg.batch, nx, nx), cov)
    assert np.array_equal(rec[:, nx + nx * nx], logc)
    assert np.all(rec[:, -1] == 0.0)


@pytest.mark.parametrize("cid, over, path", [("C5", {"batch": 3}, pmf.PATH_RESIDENT),
                                             ("C4", {"n": (32, 32, 16, 16)}, pmf.PATH_PLANE),
                                             ("C1", {}, pmf.PATH_AUTO)])
def test_checkpoint_resume(cid, over, path):
    """Checkpoint / resume through the ABI: the weights and grid of a run (pmf_get_weights,
    pmf_get_grid) loaded into a NEW context (pmf_set_state) continue the run as if it had
    not stopped."""
    cfg = make_config(cid, **over)
    T = 4
    zs = simulate(cfg, T=T)["z"]
    lik = lik_of(cfg)
    dt = cfg.tau / cfg.l

    def epochs(f, ks):
        out = []
        for k in ks:
            if k > 0:
                f.predict(dt, cfg.l)
            f.update(zs[k], lik)
            out.append(f.moments())
            f.regrid(cfg.k_sigma)
        return out

    a = make_filter(cfg, path=path)
    ra = epochs(a, range(T + 1))
    b = make_filter(cfg, path=path)
    rb = epochs(b, range(3))
    w, (c, B) = b.weights(), b.grid()                 # checkpoint after epoch 2's regrid
    b.close()
    r = pmf.Filter(cfg.nx, cfg.n, cfg.A, cfg.Q, batch=cfg.batch, path=path)
    r.set_state(c, B, w)
    rb += epochs(r, range(3, T + 1))
    for k in range(T + 1):
        for x, y in zip(ra[k][:2], rb[k][:2]):
            assert np.max(np.abs(x - y)) <= 1e-12 * max(1.0, np.max(np.abs(x))), (k, x, y)
        assert np.max(np.abs(ra[k][2] - rb[k][2])) <= 1e-12
    wa, wr = a.weights(), r.weights()
    assert rel_linf(wr, wa) <= 1e-12

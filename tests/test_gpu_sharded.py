"""The slab-sharded path: one filter split along its last axis,
two all-to-all transposes per predict, all-reduced moment sums, plane exchange at
regrid. On one GPU it runs as "virtual ranks" (the identical code path with the
collectives as device copies); parity vs the oracle and vs the unsharded run."""
import os

import numpy as np
import pytest

from oracle import pmf_oracle as O
from paper_2412_07240_b200 import pmf
from workloads import make_config, random_density, simulate

from parity_util import TOL, compare_runs, lik_of, rel_linf, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

CASES = {
    "C4s": ("C4", {"n": (8, 6, 12, 8)}, 3, (2, 4)),
    # the three-pass route (kernels_quad.cu) sharded: K1 blocks -> all-to-all -> K2 on whole
    # (j3, j2)-planes of a k0 range -> all-to-all back -> K3 on the slab
    "C4q": ("C4", {"n": (32, 32, 32, 32)}, 2, (2, 4, 8)),
    "C4q96": ("C4", {"n": (96, 96, 16, 16)}, 2, (2, 4, 8)),
    # the thinnest shards: slabs of 2 and 1 planes, k0 ranges of 2 and 1 columns (one chunk each)
    "C4q_thin": ("C4", {"n": (32, 32, 32, 32)}, 1, (16, 32)),
    "C2s": ("C2", {"n": (32, 48)}, 4, (2, 3)),
    "C3s": ("C3", {"n": (16, 12, 24)}, 3, (2, 4)),
}


@pytest.mark.parametrize("name", list(CASES))
def test_sharded_filter_run_parity(name):
    cid, over, T, worlds = CASES[name]
    cfg = make_config(cid, **over)
    zs = simulate(cfg, T=T)["z"]
    orc = run_oracle(cfg, zs, T)
    ref = run_gpu(cfg, zs, T, path=pmf.PATH_PENCIL)
    for world in worlds:
        g = run_gpu(cfg, zs, T, path=pmf.PATH_PENCIL, world=world)
        assert g["filter"].world == world
        e = compare_runs(cfg, g, orc, T, TOL["f64"])
        assert e["w"] <= 1e-10 and e["mean"] <= 1e-10 and e["cov"] <= 1e-10 and e["logC"] <= 1e-10, (world, e)
        assert e["grid"] <= 1e-10, (world, e)
        for k in range(T + 1):
            assert rel_linf(g["w"][k], ref["w"][k]) <= 1e-12, (world, k)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_predict_and_far_regrid(world):
    """Sheared grid, non-diagonal A and Q (non-separable regrid map), and a posterior
    far from the grid centre, so the new slabs read old planes owned by other ranks."""
    nx, n = 2, (32, 48)
    rng = np.random.default_rng(8)
    A = 0.5 * rng.standard_normal((nx, nx))
    M = rng.standard_normal((nx, nx))
    Q = 0.05 * (M @ M.T) + 0.02 * np.eye(nx)
    B = np.diag([0.08, 0.06]) + 0.01 * rng.standard_normal((nx, nx))
    c = np.array([0.3, -0.2])
    wlib = random_density(n, 1, seed=12)[0]
    tau, l = 0.3, 5
    H, R = np.array([[0.3, 1.0]]), np.array([[0.05]])
    z = np.array([[0.6]])
    out = []
    for w in (1, world):
        f = pmf.Filter(nx, n, A, Q, path=pmf.PATH_PENCIL, world=w, sharded=(w > 1))
        f.set_state(c[None], B[None], wlib)
        f.predict(tau / l, l)
        f.update(z, pmf.make_likelihood(pmf.LIK_LINEAR_GAUSS, nx, H=H, R=R))
        mean, cov, logc = f.moments()
        wpost = f.weights()[0]
        f.regrid(3.0)
        out.append((wpost, mean, cov, logc, f.weights()[0], f.grid()))
    # oracle
    w0 = O.normalise(O.from_lib(wlib, n), B)
    w1, c1, B1 = O.predict(w0, c, B, A, Q, tau, l)
    lk = O.lik_linear_gauss(O.grid_points(c1, B1, n), z[0], H, R)
    w2, lo = O.update(w1, c1, B1, lk)
    mo, co = O.moments(w2, c1, B1)
    c2, B2 = O.regrid_target(mo, co, n, 3.0)
    w3 = O.regrid(w2, c1, B1, c2, B2)
    for wpost, mean, cov, logc, wreg, (cg, Bg) in out:
        assert rel_linf(wpost, O.to_lib(w2)) <= 1e-10
        assert abs(logc[0] - lo) <= 1e-10 and rel_linf(mean[0], mo) <= 1e-10 and rel_linf(cov[0], co) <= 1e-10
        assert rel_linf(wreg, O.to_lib(w3)) <= 1e-10
        assert rel_linf(Bg[0], B2) <= 1e-12
    assert rel_linf(out[1][4], out[0][4]) <= 1e-12


def test_sharded_argument_errors():
    cfg = make_config("C4", n=(8, 6, 12, 8))
    with pytest.raises(pmf.PMFError):
        pmf.Filter(4, cfg.n, cfg.A, cfg.Q, world=3)            # 8 planes do not split in 3
    with pytest.raises(pmf.PMFError):
        pmf.Filter(4, cfg.n, cfg.A, cfg.Q, batch=2, world=2)   # one filter per sharded context


def test_sharded_crank_nicolson():
    """Crank-Nicolson substeps (R27) through the sharded (virtual-rank) path."""
    cfg = make_config("C4", n=(8, 6, 12, 8))
    T = 2
    zs = simulate(cfg, T=T)["z"]
    orc = {0: O.run_filter(cfg, zs, b=0, T=T, keep_weights=True, step=O.STEP_CN)}
    g = run_gpu(cfg, zs, T, path=pmf.PATH_PENCIL, world=2, step=pmf.STEP_CN)
    e = compare_runs(cfg, g, orc, T, TOL["f64"])
    assert e["w"] <= 1e-10 and e["mean"] <= 1e-10 and e["cov"] <= 1e-10 and e["logC"] <= 1e-10, e


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_three_pass_route_is_taken(world):
    """The sharded nx = 4 fp64 context runs the three-pass route (K1 blocks, two all-to-all,
    K2, K3: 5 kernels + prep/sum/finaliser per shard), not the pencil passes."""
    cfg = make_config("C4", n=(32, 32, 32, 32))
    zs = simulate(cfg, T=1)["z"]
    f = pmf.Filter(cfg.nx, cfg.n, cfg.A, cfg.Q, world=world, sharded=True)
    f.set_gaussian(cfg.prior_mean, cfg.prior_cov[None], cfg.k_sigma)
    f.update(zs[0], lik_of(cfg))
    l0 = f.launches
    f.predict(cfg.tau / cfg.l, cfg.l)
    f.sync()
    # per shard: prep, K1 and K2 in C chunks each (the pipelined all-to-alls: PMF_XCHUNKS,
    # default 4, at most slab / N0/G chunks), K3, sum, finaliser (+ the virtual all-reduce's sum)
    ch = max(1, min(16, int(os.environ.get("PMF_XCHUNKS", "4"))))
    c1, c2 = min(ch, cfg.n[3] // world), min(ch, cfg.n[0] // world)
    assert f.launches - l0 == (4 + c1 + c2) * world + 1, f.launches - l0


@pytest.mark.parametrize("name,real", [("C4q", True), ("C4q96", True), ("C3s", True), ("C2s", True),
                                       ("C4q", False), ("C3s", False)])
def test_single_rank_sharded_context(name, real):
    """real: the multi-process code path proper on one GPU -- a real NCCL communicator of world
    size 1 (pmf_nccl_unique_id + pmf_create_sharded with unique_id != NULL). libnccl is loaded,
    the communicator initialised, the all-to-all plans run (a rank's own piece is a device copy
    inside the NCCL group), the moment sums go through ncclAllReduce and
    ncclCommGetAsyncError is polled after every exchange -- none of which the virtual-rank
    contexts execute. not real: one virtual slab. G = 1 is also the degenerate case of the
    three-pass route: K2 keeps the unsharded k1-major output order, so it is not split into k0
    chunks (found by this test: the chunked K2 wrote its pieces at chunk-relative offsets).
    Parity vs the oracle."""
    cid, over, T, _ = CASES[name]
    cfg = make_config(cid, **over)
    zs = simulate(cfg, T=T)["z"]
    orc = run_oracle(cfg, zs, T)
    kw = {}
    if real:
        uid = pmf.nccl_unique_id()
        assert len(uid) == 128 and any(uid)
        kw = dict(rank=0, unique_id=uid)
    g = run_gpu(cfg, zs, T, path=pmf.PATH_PENCIL, world=1, sharded=True, **kw)
    assert g["filter"].world == 1 and g["filter"].epoch_kernel == "sharded"
    e = compare_runs(cfg, g, orc, T, TOL["f64"])
    assert e["w"] <= 1e-10 and e["mean"] <= 1e-10 and e["cov"] <= 1e-10 and e["logC"] <= 1e-10, e
    assert e["grid"] <= 1e-10, e


@pytest.mark.parametrize("name", ["C4q", "C4s", "C3s", "C2s"])
def test_sharded_step_api(name):
    """pmf_step (regrid + predict + update in one call: the call bench.py times) on sharded
    contexts -- two virtual ranks and a real 1-rank NCCL communicator -- against the unsharded
    unfused sequence: moments and normaliser of every epoch to 1e-12."""
    cid, over, T, _ = CASES[name]
    cfg = make_config(cid, **over)
    zs = simulate(cfg, T=T)["z"]
    ref = run_gpu(cfg, zs, T, path=pmf.PATH_PENCIL)
    for kw in ({"world": 2}, {"world": 1, "rank": 0, "unique_id": pmf.nccl_unique_id()}):
        g = run_gpu(cfg, zs, T, path=pmf.PATH_PENCIL, use_step=True, sharded=True, **kw)
        assert g["filter"].epoch_kernel == "sharded"
        for k in range(T + 1):
            assert np.max(np.abs(g["mean"][k] - ref["mean"][k])) <= 1e-12, (kw["world"], k)
            assert rel_linf(g["cov"][k], ref["cov"][k]) <= 1e-12, (kw["world"], k)
            assert np.max(np.abs(g["logC"][k] - ref["logC"][k])) <= 1e-12, (kw["world"], k)

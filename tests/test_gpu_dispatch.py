"""Which kernel family runs each BASELINE config's epoch (pmf_epoch_kernel), and that the
single-launch epoch kernels agree with the multi-kernel pencil path they replace when
they are switched off (PMF_NO_CLUSTER / PMF_NO_LINE_EPOCH) -- both sides also match the
oracle in test_gpu_parity.py / test_gpu_fullsize.py."""
import numpy as np
import pytest

from paper_2412_07240_b200 import pmf
from workloads import make_config, simulate

from parity_util import lik_of, make_filter, rel_linf

pytestmark = pytest.mark.gpu


def _epochs(cfg, zs, T, use_step=True, **kw):
    f = make_filter(cfg, **kw)
    lik = lik_of(cfg)
    dt = cfg.tau / cfg.l
    f.update(zs[0], lik)
    for k in range(1, T + 1):
        if use_step:
            f.step(dt, cfg.l, zs[k], lik, cfg.k_sigma)
        else:
            f.regrid(cfg.k_sigma)
            f.predict(dt, cfg.l)
            f.update(zs[k], lik)
    mean, cov, logc = f.moments()
    out = (f.epoch_kernel, f.weights(), mean, cov, logc)
    f.close()
    return out


@pytest.mark.parametrize("cid, over, want", [
    ("C1", {"batch": 3}, "line"),
    ("C2", {}, "cluster"),
    ("C5", {"batch": 4}, "resident"),
    ("C3", {}, "plane"),
    ("C4", {"n": (32, 32, 16, 16)}, "plane"),
    ("C6", {}, "pencil"),
])
def test_epoch_kernel_family(cid, over, want):
    cfg = make_config(cid, **over)
    zs = simulate(cfg, T=2)["z"]
    fam = _epochs(cfg, zs, 2)[0]
    assert fam == want, (cid, fam)


def test_epoch_kernel_fdm_and_pencil():
    cfg = make_config("C5", batch=2)
    zs = simulate(cfg, T=1)["z"]
    assert _epochs(cfg, zs, 1, diff_mode=pmf.DIFF_FDM)[0] == "fdm"
    assert _epochs(cfg, zs, 1, path=pmf.PATH_PENCIL)[0] == "pencil"


@pytest.mark.parametrize("cid, over, env", [("C2", {}, "PMF_NO_CLUSTER"),
                                            ("C1", {"batch": 5}, "PMF_NO_LINE_EPOCH")])
def test_single_launch_epoch_matches_multi_kernel(cid, over, env, monkeypatch):
    cfg = make_config(cid, **over)
    T = 4
    zs = simulate(cfg, T=T)["z"]
    fam_a, w_a, m_a, c_a, l_a = _epochs(cfg, zs, T)
    monkeypatch.setenv(env, "1")
    fam_b, w_b, m_b, c_b, l_b = _epochs(cfg, zs, T)
    assert fam_a != "pencil" and fam_b == "pencil"
    assert rel_linf(w_a, w_b) <= 1e-11
    assert np.max(np.abs(m_a - m_b)) <= 1e-11 * (1 + np.max(np.abs(m_b)))
    assert np.max(np.abs(c_a - c_b)) <= 1e-11 * np.max(np.abs(c_b))
    assert np.max(np.abs(l_a - l_b)) <= 1e-10

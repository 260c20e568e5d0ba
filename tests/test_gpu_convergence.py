"""NEXT-2: the paper's time-update convergence experiment (Figs. 1-3) on
the GPU (tools/convergence.py): the orderings the paper states, on the GPU results,
plus GPU == oracle on one case of each predictor. The figures print no numbers, so
only orderings and orders are checked."""
import importlib.util
import os

import numpy as np
import pytest

from oracle import pmf_oracle as O

pytestmark = pytest.mark.gpu

_spec = importlib.util.spec_from_file_location(
    "convergence", os.path.join(os.path.dirname(os.path.dirname(__file__)), "tools", "convergence.py"))
conv = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(conv)


@pytest.mark.parametrize("name", ["gauss", "gm3"])
def test_orderings(name):
    from paper_2412_07240_b200 import pmf
    comps = conv.DENSITIES[name]
    fdm = {N: conv.run(N, comps, pmf.DIFF_FDM, 64) for N in (32, 64, 128)}
    spec = {N: conv.run(N, comps, pmf.DIFF_FULL, 1000) for N in (32, 64, 96)}
    order = np.log(fdm[32] / fdm[128]) / np.log(4.0)
    assert 1.7 < order < 2.4, fdm                       # FDM: O(1/N^2)
    assert spec[64] < 0.1 * fdm[64], (spec, fdm)         # spectral >> FDM at equal N
    assert spec[96] < 0.05 * fdm[128], (spec, fdm)      # (spectral floor: its Euler time error)


@pytest.mark.parametrize("mode", ["spectral", "fdm"])
def test_gpu_matches_oracle(mode):
    from paper_2412_07240_b200 import pmf
    comps = conv.DENSITIES["gm3"]
    N = 64
    mu, sd = conv.extent(comps)
    delta = 16.0 * sd / N
    c, B = np.array([mu]), np.array([[delta]])
    x = mu + delta * (np.arange(N) - (N - 1) / 2.0)
    w = conv.mixture(x, comps)
    w = w / (w.sum() * delta)
    l = 64
    dm = pmf.DIFF_FULL if mode == "spectral" else pmf.DIFF_FDM
    f = pmf.Filter(1, (N,), np.zeros((1, 1)), np.array([[conv.Q]]), diff_mode=dm)
    f.set_state(c[None], B[None], w)
    f.predict(conv.TAU / l, l)
    g = f.weights()[0]
    o, _, _ = O.predict(w, c, B, np.zeros((1, 1)), np.array([[conv.Q]]), conv.TAU, l,
                        diff_mode=O.DIFF_FULL if mode == "spectral" else O.DIFF_FDM)
    assert float(np.max(np.abs(g - o)) / np.max(np.abs(o))) < 1e-12

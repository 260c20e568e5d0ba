import numpy as np, sys
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), 'tests'))
from paper_2412_07240_b200 import pmf
from workloads import make_config, simulate
from parity_util import lik_of
for cid, n in (("C3", (32, 32, 32)), ("C3", (64, 64, 16)), ("C3", (32, 32, 64))):
    cfg = make_config(cid, n=n)
    zs = simulate(cfg, T=2)["z"]
    res = {}
    for path in (pmf.PATH_PLANE, pmf.PATH_PENCIL):
        f = pmf.Filter(cfg.nx, cfg.n, cfg.A, cfg.Q, path=path)
        f.set_gaussian(cfg.prior_mean, cfg.prior_cov[None], cfg.k_sigma)
        f.predict(cfg.tau / cfg.l, cfg.l)
        w1 = f.weights()[0]
        lik = lik_of(cfg)
        try:
            f.update(zs[1], lik)
            w2 = f.weights()[0]; mom = f.moments()
        except Exception as e:
            w2 = None; mom = str(e)
        res[path] = (w1, w2, mom)
    a, b = res[pmf.PATH_PLANE], res[pmf.PATH_PENCIL]
    print(cid, n, "predict err", float(np.max(np.abs(a[0] - b[0])) / np.max(np.abs(b[0]))), "nan?", np.isnan(a[0]).any())
    if a[1] is not None:
        print("   update err", float(np.max(np.abs(a[1] - b[1])) / np.max(np.abs(b[1]))), a[2][2], b[2][2])
    else:
        print("   update failed", a[2])

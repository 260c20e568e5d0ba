import os, sys
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, 'tests'))
import numpy as np
from oracle import pmf_oracle as O
from paper_2412_07240_b200 import pmf
from workloads import make_config, simulate
from parity_util import lik_of
cfg = make_config("C1", n=(32,))
zs = simulate(cfg, T=5)["z"]
orc = O.run_filter(cfg, zs, b=0, T=5, keep_weights=True, diff_mode=O.DIFF_FDM)
f = pmf.Filter(1, (32,), cfg.A, cfg.Q, diff_mode=pmf.DIFF_FDM)
f.set_gaussian(cfg.prior_mean, cfg.prior_cov[None], cfg.k_sigma)
lik = lik_of(cfg)
for k in range(6):
    try:
        if k > 0:
            f.predict(cfg.tau / cfg.l, cfg.l)
            print(k, "pred w", f.weights()[0][:4], f.grid())
        f.update(zs[k], lik)
        m, c, lc = f.moments()
        print(k, m, orc["mean"][k], lc, orc["logC"][k])
        f.regrid(cfg.k_sigma)
    except Exception as e:
        print(k, "ERR", e); break

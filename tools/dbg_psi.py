import os, sys
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R)
import numpy as np
from paper_2412_07240_b200 import pmf
from workloads import random_density
n = (64, 64, 16)
rng = np.random.default_rng(1)
for l in (1, 2, 3, 4):
    for Qd in ((0.1, 0.1, 0.1), (0.0, 0.0, 0.1), (0.1, 0.0, 0.0)):
        A = np.zeros((3, 3)); Q = np.diag(Qd)
        B = np.diag([0.05, 0.05, 0.1]); c = np.zeros(3)
        w = random_density(n, 1, seed=3)[0]
        outs = []
        for path in (pmf.PATH_PLANE, pmf.PATH_PENCIL):
            f = pmf.Filter(3, n, A, Q, path=path)
            f.set_state(c[None], B[None], w)
            f.predict(0.1 / l, l)
            outs.append(f.weights()[0])
        e = float(np.max(np.abs(outs[0] - outs[1])) / np.max(np.abs(outs[1])))
        print(l, Qd, f"{e:.3e}")

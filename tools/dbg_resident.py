import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from workloads import make_config, simulate
from paper_2412_07240_b200 import pmf
from parity_util import run_gpu
cfg = make_config("C5", batch=3)
zs = simulate(cfg, T=2)["z"]
try:
    a = run_gpu(cfg, zs, 2, path=pmf.PATH_RESIDENT)
    print("ok")
except Exception as e:
    print("EXC", e)

"""B200-native spectral point-mass filter (arXiv 2412.07240) hot path.

The product is libpmf.so (C ABI, include/pmf.h) built from csrc/ for sm_100a;
``paper_2412_07240_b200.pmf`` is its thin ctypes binding.
"""
from .pmf import Filter, PMFError, load_library, make_likelihood  # noqa: F401

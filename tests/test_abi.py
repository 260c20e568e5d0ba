"""CPU checks of the C-ABI boundary: libpmf.so builds/loads, exports every
symbol include/pmf.h declares, and validates arguments before touching a GPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2412_07240_b200 import pmf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "pmf.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(pmf_[a-z_0-9]+)\s*\(", txt)))


def test_header_symbols_exported():
    lib = pmf.load_library()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(pmf.SYMBOLS) == syms


def _create(nx, n, A, Q, **kw):
    lib = pmf.load_library()
    cfg = pmf.pmf_config()
    cfg.nx = nx
    for i, v in enumerate(n):
        cfg.n[i] = v
    cfg.batch = kw.get("batch", 1)
    cfg.dtype = kw.get("dtype", 0)
    cfg.diff_mode = kw.get("diff_mode", 0)
    cfg.grid = kw.get("grid", 0)
    h = C.c_void_p()
    A = np.ascontiguousarray(np.asarray(A, dtype=np.float64))
    Q = np.ascontiguousarray(np.asarray(Q, dtype=np.float64))
    rc = lib.pmf_create(C.byref(cfg), pmf._dptr(A), pmf._dptr(Q), C.byref(h))
    return rc, lib.pmf_last_error(None).decode()


def test_argument_validation_without_gpu():
    eye = np.eye(2)
    assert _create(2, (31, 32), eye, eye)[0] == -2          # PMF_E_ODD_N
    assert _create(2, (38, 32), eye, eye)[0] == -3          # PMF_E_RADIX (38 = 2 x 19)
    assert _create(2, (2048, 32), eye, eye)[0] == -3        # too large
    assert _create(5, (8,), np.eye(5), np.eye(5))[0] == -1  # nx range
    assert _create(2, (8, 8), eye, np.array([[1.0, 0.0], [0.5, 1.0]]))[0] == -4   # not symmetric
    assert _create(2, (8, 8), eye, np.diag([1.0, -1.0]))[0] == -4               # not PSD
    assert _create(2, (8, 8), eye, np.array([[1.0, 0.2], [0.2, 1.0]]), diff_mode=1)[0] == -1
    assert _create(1, (8,), [[0.0]], [[1.0]], dtype=7)[0] == -1
    assert _create(2, (8, 8), eye, eye, grid=5)[0] == -1                               # bad grid policy
    assert _create(2, (32, 32), eye, eye, grid=pmf.GRID_EIGEN, diff_mode=2)[0] == -1    # eigen grid + FDM


def test_no_cpu_fallback():
    """Without a usable CUDA device creation fails loudly (PMF_E_CUDA)."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    rc, msg = _create(1, (64,), [[-0.5]], [[1.0]])
    assert rc == -9 and "no CPU fallback" in msg
    with pytest.raises(pmf.PMFError):
        pmf.Filter(1, (64,), [[-0.5]], [[1.0]])


def _header_defines(prefix):
    txt = open(os.path.join(ROOT, "include", "pmf.h")).read()
    return {m[0]: int(m[1]) for m in re.findall(rf"#define\s+({prefix}[A-Z_0-9]+)\s+(-?\d+)", txt)}


def test_binding_constants_match_header():
    """The binding's constants are the header's (the ctypes layer has no other source)."""
    ep = _header_defines("PMF_EPOCH_")
    assert {v: k[len("PMF_EPOCH_"):].lower() for k, v in ep.items()} == pmf.EPOCH_KERNELS
    paths = _header_defines("PMF_PATH_")
    assert (paths["PMF_PATH_AUTO"], paths["PMF_PATH_PENCIL"], paths["PMF_PATH_RESIDENT"],
            paths["PMF_PATH_PLANE"]) == (pmf.PATH_AUTO, pmf.PATH_PENCIL, pmf.PATH_RESIDENT, pmf.PATH_PLANE)
    errs = _header_defines("PMF_E_")
    assert {v: k for k, v in errs.items()} == pmf.ERRORS
    grids = _header_defines("PMF_GRID_")
    assert (grids["PMF_GRID_AXIS"], grids["PMF_GRID_EIGEN"]) == (pmf.GRID_AXIS, pmf.GRID_EIGEN)
    lib = pmf.load_library()
    assert lib.pmf_epoch_kernel(None) == -1 and lib.pmf_path(None) == -1


def test_binding_validates_buffers():
    """Raw pointers are only taken from buffers of the right device, dtype, layout and size
    (ADVICE r1): a CPU tensor never reaches the library as a device pointer, and host
    output arrays must be float64, C-contiguous and of the exact shape."""
    import torch
    with pytest.raises(pmf.PMFError):
        pmf._check_device_tensor(torch.zeros(8, dtype=torch.float64), 0, torch.float64, 8, "x")
    pmf._check_host_array(np.zeros((3, 2)), (3, 2), "mean")
    for bad in (np.zeros((3, 2), dtype=np.float32), np.zeros((2, 3)).T, np.zeros((3, 3)), [[0.0] * 2] * 3):
        with pytest.raises(pmf.PMFError):
            pmf._check_host_array(bad, (3, 2), "mean")

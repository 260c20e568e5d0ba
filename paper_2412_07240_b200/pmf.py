"""Thin ctypes binding of libpmf.so (include/pmf.h): argument marshalling only.

Every step of the filter runs in the library's CUDA kernels; this module only
packs arrays, passes torch's CUDA stream and device pointers, and raises
``PMFError`` on non-zero return codes. There is no CPU fallback: importing
works anywhere, but creating a ``Filter`` needs libpmf.so and a CUDA device.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PMF_LIB") or os.path.join(_HERE, "libpmf.so")   # PMF_LIB: A/B builds (tools/ab.sh)

PMF_OK = 0
ERRORS = {-1: "PMF_E_ARG", -2: "PMF_E_ODD_N", -3: "PMF_E_RADIX", -4: "PMF_E_Q_NOT_PSD",
          -5: "PMF_E_SINGULAR_GRID", -6: "PMF_E_NO_SUPPORT", -7: "PMF_E_DT", -8: "PMF_E_STATE",
          -9: "PMF_E_CUDA", -10: "PMF_E_NOMEM", -11: "PMF_E_NCCL"}
F64, F32 = 0, 1
DIFF_FULL, DIFF_AXIS_LITERAL, DIFF_FDM = 0, 1, 2
STEP_EULER, STEP_CN = 0, 1
GRID_AXIS, GRID_EIGEN = 0, 1   # grid design from a covariance: axis-aligned (R12) / eigenvector-aligned (R28)
TRACE_PHYSICAL, TRACE_PRINTED = -1, 1
PATH_AUTO, PATH_PENCIL, PATH_RESIDENT, PATH_PLANE = 0, 1, 2, 3
# kernel family of the last predict (pmf_epoch_kernel)
EPOCH_KERNELS = {0: "none", 1: "pencil", 2: "line", 3: "cluster", 4: "resident", 5: "plane", 6: "fdm",
                 7: "sharded"}
LIK_LINEAR_GAUSS, LIK_RANGE_GAUSS, LIK_TERRAIN_GM = 0, 1, 2

# every symbol include/pmf.h declares (checked by tests/test_abi.py)
SYMBOLS = ["pmf_create", "pmf_destroy", "pmf_last_error", "pmf_set_gaussian", "pmf_set_state",
           "pmf_predict", "pmf_update", "pmf_moments", "pmf_regrid", "pmf_step", "pmf_get_weights",
           "pmf_get_grid", "pmf_sync", "pmf_launch_count", "pmf_moments_bytes", "pmf_nccl_unique_id",
           "pmf_create_sharded", "pmf_world", "pmf_profile", "pmf_profile_read", "pmf_use_graphs",
           "pmf_set_terrain", "pmf_device_bytes", "pmf_path", "pmf_version", "pmf_moments_async",
           "pmf_epoch_kernel"]


class PMFError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class pmf_config(C.Structure):
    _fields_ = [("nx", C.c_int), ("n", C.c_int * 4), ("batch", C.c_int), ("dtype", C.c_int),
                ("diff_mode", C.c_int), ("trace_sign", C.c_int), ("path", C.c_int), ("device", C.c_int),
                ("stream", C.c_void_p), ("step", C.c_int), ("grid", C.c_int)]


class pmf_likelihood(C.Structure):
    _fields_ = [("kind", C.c_int), ("nz", C.c_int), ("H", C.c_double * 16), ("R", C.c_double * 16),
                ("sigma", C.c_double), ("ncomp", C.c_int), ("gm_w", C.c_double * 4), ("gm_mu", C.c_double * 4),
                ("gm_var", C.c_double * 4)]


_lib = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load libpmf.so; raises (loudly) if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libpmf.so not built at {path}: run `python -m paper_2412_07240_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(path)
    P, D, I, V = C.c_void_p, C.POINTER(C.c_double), C.c_int, C.c_void_p
    sig = {
        "pmf_create": (I, [C.POINTER(pmf_config), D, D, C.POINTER(P)]),
        "pmf_destroy": (None, [P]),
        "pmf_last_error": (C.c_char_p, [P]),
        "pmf_set_gaussian": (I, [P, D, D, C.c_double]),
        "pmf_set_state": (I, [P, D, D, V, I]),
        "pmf_predict": (I, [P, C.c_double, I]),
        "pmf_update": (I, [P, V, I, C.POINTER(pmf_likelihood)]),
        "pmf_moments": (I, [P, D, D, D]),
        "pmf_regrid": (I, [P, C.c_double]),
        "pmf_step": (I, [P, C.c_double, I, V, I, C.POINTER(pmf_likelihood), C.c_double]),
        "pmf_get_weights": (I, [P, V, I]),
        "pmf_get_grid": (I, [P, D, D]),
        "pmf_sync": (I, [P]),
        "pmf_launch_count": (C.c_int64, [P]),
        "pmf_moments_bytes": (C.c_int64, [P]),
        "pmf_moments_async": (I, [P, V]),
        "pmf_nccl_unique_id": (I, [V]),
        "pmf_create_sharded": (I, [C.POINTER(pmf_config), D, D, I, I, V, C.POINTER(P)]),
        "pmf_world": (I, [P]),
        "pmf_profile": (I, [P, I]),
        "pmf_use_graphs": (I, [P, I]),
        "pmf_set_terrain": (I, [P, D, I, I, C.c_double, C.c_double, C.c_double, C.c_double, I, I]),
        "pmf_profile_read": (I, [P, C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
        "pmf_device_bytes": (C.c_int64, [P]),
        "pmf_path": (I, [P]),
        "pmf_epoch_kernel": (I, [P]),
        "pmf_version": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def nccl_unique_id() -> bytes:
    """128-byte NCCL id for pmf_create_sharded (create on rank 0, broadcast to the others)."""
    lib = load_library()
    buf = C.create_string_buffer(128)
    rc = lib.pmf_nccl_unique_id(buf)
    if rc != PMF_OK:
        raise PMFError(rc, lib.pmf_last_error(None).decode())
    return buf.raw


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _arg_error(msg: str) -> PMFError:
    return PMFError(-1, msg)


def _check_device_tensor(t, device: int, dtype, min_numel: int, what: str):
    """A torch tensor handed to the library as a raw device pointer: it must live on the
    context's CUDA device, have the expected dtype, be contiguous and hold at least
    min_numel elements -- anything else would be read or written out of bounds."""
    if not getattr(t, "is_cuda", False):
        raise _arg_error(f"{what}: expected a CUDA tensor on cuda:{device}, got device {getattr(t, 'device', '?')}")
    if t.device.index != device:
        raise _arg_error(f"{what}: tensor is on cuda:{t.device.index}, the filter on cuda:{device}")
    if t.dtype != dtype:
        raise _arg_error(f"{what}: dtype {t.dtype}, expected {dtype}")
    if not t.is_contiguous():
        raise _arg_error(f"{what}: tensor must be contiguous")
    if t.numel() < min_numel:
        raise _arg_error(f"{what}: {t.numel()} elements, need {min_numel}")


def _check_host_array(a, shape, what: str):
    """A numpy array the library writes into: float64, C-contiguous, exactly `shape`."""
    if not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags.c_contiguous or \
            tuple(a.shape) != tuple(shape):
        raise _arg_error(f"{what}: need a C-contiguous float64 array of shape {tuple(shape)}")


def make_likelihood(kind: int, nx: int, H=None, R=None, sigma: float = 0.0, gm=None) -> pmf_likelihood:
    """gm (TERRAIN_GM): sequence of (weight, mean, variance) noise components."""
    lk = pmf_likelihood()
    lk.kind = kind
    if kind == LIK_TERRAIN_GM:
        lk.nz = 1
        lk.ncomp = len(gm)
        for g, (w, mu, var) in enumerate(gm):
            lk.gm_w[g], lk.gm_mu[g], lk.gm_var[g] = float(w), float(mu), float(var)
        return lk
    if kind == LIK_RANGE_GAUSS:
        lk.nz = 1
        lk.sigma = float(sigma)
    else:
        H = np.atleast_2d(np.asarray(H, dtype=np.float64))
        R = np.atleast_2d(np.asarray(R, dtype=np.float64))
        lk.nz = H.shape[0]
        for i, v in enumerate(H.reshape(-1)):
            lk.H[i] = v
        for i, v in enumerate(R.reshape(-1)):
            lk.R[i] = v
    return lk


class Filter:
    """A batch of spectral point-mass filters on the GPU (one pmf_ctx)."""

    def __init__(self, nx: int, n, A, Q, batch: int = 1, dtype: str = "f64", diff_mode: int = DIFF_FULL,
                 trace_sign: int = TRACE_PHYSICAL, path: int = PATH_AUTO, device: int = 0,
                 stream: Optional[int] = None, world: int = 1, rank: int = 0,
                 unique_id: Optional[bytes] = None, sharded: bool = False, step: int = STEP_EULER,
                 grid: int = GRID_AXIS):
        """world > 1 (or sharded=True): one filter split into `world` slabs along the last
        axis -- with `unique_id` (from nccl_unique_id(), broadcast to all ranks) this
        process is `rank` over NCCL; without it all slabs are "virtual ranks" here."""
        self.lib = load_library()
        self.nx, self.n, self.batch = nx, tuple(int(v) for v in n), batch
        self.device = int(device)
        self.dtype = dtype
        self.np_dtype = np.float64 if dtype == "f64" else np.float32
        cfg = pmf_config()
        cfg.nx = nx
        for i in range(4):
            cfg.n[i] = self.n[i] if i < nx else 1
        cfg.batch = batch
        cfg.dtype = F64 if dtype == "f64" else F32
        cfg.diff_mode = diff_mode
        cfg.trace_sign = trace_sign
        cfg.path = path
        cfg.device = device
        cfg.step = step
        cfg.grid = grid
        if stream is None:
            try:
                import torch
                if torch.cuda.is_available():
                    stream = torch.cuda.current_stream(device).cuda_stream
            except Exception:
                stream = None
        cfg.stream = C.c_void_p(stream) if stream else None
        A = np.ascontiguousarray(np.asarray(A, dtype=np.float64).reshape(nx, nx))
        Q = np.ascontiguousarray(np.asarray(Q, dtype=np.float64).reshape(nx, nx))
        h = C.c_void_p()
        if world > 1 or sharded:
            uid = C.create_string_buffer(bytes(unique_id), 128) if unique_id is not None else None
            rc = self.lib.pmf_create_sharded(C.byref(cfg), _dptr(A), _dptr(Q), int(rank), int(world),
                                             uid, C.byref(h))
        else:
            rc = self.lib.pmf_create(C.byref(cfg), _dptr(A), _dptr(Q), C.byref(h))
        if rc != PMF_OK:
            raise PMFError(rc, self.lib.pmf_last_error(None).decode())
        self.h = h
        self.ntot = int(np.prod(self.n))

    # --------------------------------------------------------------- helpers
    def _check(self, rc: int):
        if rc != PMF_OK:
            raise PMFError(rc, self.lib.pmf_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            self.lib.pmf_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --------------------------------------------------------------- ABI
    def set_gaussian(self, mean, cov, k_sigma: float):
        mean = np.ascontiguousarray(np.broadcast_to(np.asarray(mean, dtype=np.float64),
                                                    (self.batch, self.nx)))
        cov = np.ascontiguousarray(np.broadcast_to(np.asarray(cov, dtype=np.float64),
                                                   (self.batch, self.nx, self.nx)))
        self._check(self.lib.pmf_set_gaussian(self.h, _dptr(mean), _dptr(cov), float(k_sigma)))

    def set_state(self, center, B, weights):
        center = np.ascontiguousarray(np.asarray(center, dtype=np.float64).reshape(self.batch, self.nx))
        B = np.ascontiguousarray(np.asarray(B, dtype=np.float64).reshape(self.batch, self.nx, self.nx))
        if hasattr(weights, "data_ptr"):      # torch tensor on the device
            _check_device_tensor(weights, self.device, self._torch_dtype(), self.batch * self.ntot, "set_state weights")
            self._check(self.lib.pmf_set_state(self.h, _dptr(center), _dptr(B), C.c_void_p(weights.data_ptr()), 1))
        else:
            w = np.ascontiguousarray(np.asarray(weights, dtype=self.np_dtype).reshape(-1))
            self._check(self.lib.pmf_set_state(self.h, _dptr(center), _dptr(B), w.ctypes.data_as(C.c_void_p), 0))

    def predict(self, dt: float, steps: int):
        self._check(self.lib.pmf_predict(self.h, float(dt), int(steps)))

    def _torch_dtype(self):
        import torch
        return torch.float64 if self.dtype == "f64" else torch.float32

    def _z(self, z, lik: pmf_likelihood):
        need = self.batch * int(lik.nz)
        if hasattr(z, "data_ptr"):
            if getattr(z, "is_cuda", False):
                import torch
                _check_device_tensor(z, self.device, torch.float64, need, "z")
                return C.c_void_p(z.data_ptr()), 1, z
            z = z.numpy()                     # a CPU tensor: passed as host memory
        zz = np.ascontiguousarray(np.asarray(z, dtype=np.float64).reshape(-1))
        if zz.size < need:
            raise _arg_error(f"z: {zz.size} values, need batch x nz = {need}")
        return zz.ctypes.data_as(C.c_void_p), 0, zz

    def update(self, z, lik: pmf_likelihood):
        p, dev, keep = self._z(z, lik)
        self._check(self.lib.pmf_update(self.h, p, dev, C.byref(lik)))
        del keep

    def regrid(self, k_sigma: float):
        self._check(self.lib.pmf_regrid(self.h, float(k_sigma)))

    def step(self, dt: float, steps: int, z, lik: pmf_likelihood, k_sigma: float):
        p, dev, keep = self._z(z, lik)
        self._check(self.lib.pmf_step(self.h, float(dt), int(steps), p, dev, C.byref(lik), float(k_sigma)))
        del keep

    def moments(self):
        mean = np.empty((self.batch, self.nx))
        cov = np.empty((self.batch, self.nx, self.nx))
        logc = np.empty(self.batch)
        self._check(self.lib.pmf_moments(self.h, _dptr(mean), _dptr(cov), _dptr(logc)))
        return mean, cov, logc

    def moments_into(self, mean: np.ndarray, cov: np.ndarray, logc: np.ndarray):
        _check_host_array(mean, (self.batch, self.nx), "mean")
        _check_host_array(cov, (self.batch, self.nx, self.nx), "cov")
        _check_host_array(logc, (self.batch,), "logc")
        self._check(self.lib.pmf_moments(self.h, _dptr(mean), _dptr(cov), _dptr(logc)))

    def weights(self) -> np.ndarray:
        """Normalised densities, shape (batch, N_{nx-1}, ..., N_0) (axis 0 fastest)."""
        out = np.empty((self.batch,) + tuple(reversed(self.n)), dtype=self.np_dtype)
        self._check(self.lib.pmf_get_weights(self.h, out.ctypes.data_as(C.c_void_p), 0))
        return out

    def weights_to(self, tensor):
        """Write the normalised densities into a device tensor (torch)."""
        _check_device_tensor(tensor, self.device, self._torch_dtype(), self.batch * self.ntot, "weights_to")
        self._check(self.lib.pmf_get_weights(self.h, C.c_void_p(tensor.data_ptr()), 1))

    def grid(self):
        c = np.empty((self.batch, self.nx))
        B = np.empty((self.batch, self.nx, self.nx))
        self._check(self.lib.pmf_get_grid(self.h, _dptr(c), _dptr(B)))
        return c, B

    def sync(self):
        self._check(self.lib.pmf_sync(self.h))

    @property
    def world(self) -> int:
        return int(self.lib.pmf_world(self.h))

    @property
    def launches(self) -> int:
        return int(self.lib.pmf_launch_count(self.h))

    def set_terrain(self, heights, x0: float, y0: float, dx: float, dy: float, ix: int, iy: int):
        """Terrain table for LIK_TERRAIN_GM: heights[r, c] at (x0 + c dx, y0 + r dy)."""
        h = np.ascontiguousarray(np.asarray(heights, dtype=np.float64))
        self._check(self.lib.pmf_set_terrain(self.h, _dptr(h), int(h.shape[0]), int(h.shape[1]), float(x0),
                                             float(y0), float(dx), float(dy), int(ix), int(iy)))

    def use_graphs(self, enable: bool = True):
        """CUDA-graph replay of repeated flushes (needs a non-default stream)."""
        self._check(self.lib.pmf_use_graphs(self.h, 1 if enable else 0))

    def profile(self, enable: bool = True):
        self._check(self.lib.pmf_profile(self.h, 1 if enable else 0))

    def profile_read(self):
        """(total kernel milliseconds, number of timed launches) since profile(True); syncs."""
        ms, n = C.c_double(), C.c_int64()
        self._check(self.lib.pmf_profile_read(self.h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def moments_async(self, dst) -> None:
        """Enqueue the last update's moments into ``dst`` (pinned host memory, a torch tensor
        or numpy array of moments_bytes bytes): records of (nx + nx^2 + 2) doubles per
        filter -- mean, cov, log normaliser, failure flag. Read after sync()."""
        need = self.moments_bytes
        if hasattr(dst, "data_ptr"):
            import torch
            if dst.is_cuda or dst.dtype != torch.float64 or not dst.is_contiguous() or \
                    dst.numel() * 8 < need:
                raise _arg_error(f"moments_async: need a contiguous float64 host tensor of >= {need} bytes")
            ptr = dst.data_ptr()
        else:
            if not isinstance(dst, np.ndarray) or dst.dtype != np.float64 or not dst.flags.c_contiguous or \
                    dst.nbytes < need:
                raise _arg_error(f"moments_async: need a C-contiguous float64 array of >= {need} bytes")
            ptr = dst.ctypes.data
        self._check(self.lib.pmf_moments_async(self.h, C.c_void_p(ptr)))

    @property
    def moments_bytes(self) -> int:
        return int(self.lib.pmf_moments_bytes(self.h))

    @property
    def device_bytes(self) -> int:
        return int(self.lib.pmf_device_bytes(self.h))

    @property
    def path(self) -> int:
        return int(self.lib.pmf_path(self.h))

    @property
    def epoch_kernel(self) -> str:
        """Kernel family that ran the last predict ("resident", "cluster", "line", ...)."""
        return EPOCH_KERNELS[int(self.lib.pmf_epoch_kernel(self.h))]

"""CPU test of the sharded three-pass route's slab / all-to-all offset math (no GPU): the
library's exchange plans (pmf_debug_quad_plan, the same code sh_predict_quad uses) applied to
numpy buffers laid out as the kernels write them must hand K2 whole (j3, j2)-planes of its
k0 range and K3 every (k1, k0) of its slab's planes -- each element exactly once, for
G = 1..8 ranks (slab over j3, k0 ranges for the axis-2/3 pass)."""
import ctypes as C

import numpy as np
import pytest

from paper_2412_07240_b200 import pmf


def _plan(world, blk):
    lib = pmf.load_library()
    f = lib.pmf_debug_quad_plan
    f.restype = C.c_int
    f.argtypes = [C.c_int, C.c_longlong, C.POINTER(C.c_longlong)]
    out = np.zeros(2 * world * world * 5, dtype=np.int64)
    assert f(world, blk, out.ctypes.data_as(C.POINTER(C.c_longlong))) == 0
    p = out.reshape(2, world * world, 5)
    return p[0], p[1]


def _apply(plan, send, recv):
    """Exchange: bytes -> complex (16 B) element offsets."""
    for src, dst, so, do, nb in plan:
        so, do, n = so // 16, do // 16, nb // 16
        recv[dst][do:do + n] = send[src][so:so + n]


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_three_pass_exchange_plans(world):
    N, NQ = 24, 8                          # k0 range N, H = N/2 + 1 rows k1, n2 = n3 = NQ
    H = N // 2 + 1
    if N % world or NQ % world:
        pytest.skip("sizes not divisible")
    slab, N0c = NQ // world, N // world
    rng = np.random.default_rng(world)
    S = rng.standard_normal((N, H, NQ, NQ)) + 1j * rng.standard_normal((N, H, NQ, NQ))   # S[k0, k1, j2, j3]
    blk = slab * NQ * H * N0c
    x1, x2 = _plan(world, blk)
    assert len(x1) == len(x2) == world * world
    # K1 of rank r: block q = [j3 % slab][j2][k1][k0 - q N0c] of its slab
    A = []
    for r in range(world):
        a = np.empty(world * blk, dtype=complex)
        for q in range(world):
            blkv = S[q * N0c:(q + 1) * N0c, :, :, r * slab:(r + 1) * slab]       # (k0l, k1, j2, j3l)
            a[q * blk:(q + 1) * blk] = blkv.transpose(3, 2, 1, 0).reshape(-1)
        A.append(a)
    R = [np.full(world * blk, np.nan + 0j) for _ in range(world)]
    _apply(x1, A, R)
    for q in range(world):
        assert not np.isnan(R[q].real).any()                                  # every slot filled once
        view = R[q].reshape(NQ, NQ, H, N0c)                                   # K2's map: [j3][j2][k1][k0l]
        want = S[q * N0c:(q + 1) * N0c].transpose(3, 2, 1, 0)
        assert np.array_equal(view, want)
    # K2 of rank q (identity here): output row j3 to block j3 // slab = [k0l][k1][j3 % slab][j2]
    O = []
    for q in range(world):
        view = R[q].reshape(NQ, NQ, H, N0c)
        o = np.empty(world * blk, dtype=complex)
        for r in range(world):
            part = view[r * slab:(r + 1) * slab]                              # (j3l, j2, k1, k0l)
            o[r * blk:(r + 1) * blk] = part.transpose(3, 2, 0, 1).reshape(-1)
        O.append(o)
    T = [np.full(world * blk, np.nan + 0j) for _ in range(world)]
    _apply(x2, O, T)
    for r in range(world):
        assert not np.isnan(T[r].real).any()
        view = T[r].reshape(N, H, slab, NQ)                                   # K3's map: [k0][k1][j3l][j2]
        want = S[:, :, :, r * slab:(r + 1) * slab].transpose(0, 1, 3, 2)
        assert np.array_equal(view, want)

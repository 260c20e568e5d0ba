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


def _chunk(world, blk, which, inner, lo, hi):
    lib = pmf.load_library()
    f = lib.pmf_debug_quad_chunk
    f.restype = C.c_int
    f.argtypes = [C.c_int, C.c_longlong, C.c_int, C.c_longlong, C.c_int, C.c_int, C.POINTER(C.c_longlong)]
    out = np.zeros(world * world * 5, dtype=np.int64)
    assert f(world, blk, which, inner, lo, hi, out.ctypes.data_as(C.POINTER(C.c_longlong))) == 0
    return out.reshape(world * world, 5)


@pytest.mark.parametrize("world,chunks", [(1, 3), (2, 2), (2, 4), (4, 3), (8, 4)])
def test_pipelined_exchange_chunks(world, chunks):
    """The pipelined exchanges (sh_predict_quad, PMF_XCHUNKS): K1 runs over j3 chunks
    [slab i / C, slab (i+1) / C) of its slab and chunk i's pieces leave before later rows exist;
    K2 runs over k0 chunks and chunk i returns before later k0 exist. Rows not yet computed
    are NaN in the senders: every receiver slot must still end up filled, exactly once, with
    the right element -- i.e. no piece reads ahead of its pass."""
    N, NQ = 24, 8
    H = N // 2 + 1
    slab, N0c = NQ // world, N // world
    C1, C2 = min(chunks, slab), min(chunks, N0c)
    rng = np.random.default_rng(10 * world + chunks)
    S = rng.standard_normal((N, H, NQ, NQ)) + 1j * rng.standard_normal((N, H, NQ, NQ))
    blk = slab * NQ * H * N0c
    inner1, inner2 = NQ * H * N0c, H * slab * NQ
    full = []
    for r in range(world):
        a = np.empty(world * blk, dtype=complex)
        for q in range(world):
            a[q * blk:(q + 1) * blk] = S[q * N0c:(q + 1) * N0c, :, :, r * slab:(r + 1) * slab].transpose(3, 2, 1, 0).reshape(-1)
        full.append(a)
    R = [np.full(world * blk, np.nan + 0j) for _ in range(world)]
    nbytes = 0
    for i in range(C1):
        jb, je = slab * i // C1, slab * (i + 1) // C1
        partial = []
        for r in range(world):                     # K1 has written rows j3 % slab < je only
            a = np.full(world * blk, np.nan + 0j)
            for q in range(world):
                lo = q * blk
                a[lo:lo + je * inner1] = full[r][lo:lo + je * inner1]
            partial.append(a)
        pc = _chunk(world, blk, 0, inner1, jb, je)
        for src, dst, so, do, nb in pc:
            assert np.isnan(R[dst][do // 16:(do + nb) // 16].real).all()   # each slot written once
        _apply(pc, partial, R)
        nbytes += int(pc[:, 4].sum())
    assert nbytes == 16 * world * world * blk
    for q in range(world):
        assert np.array_equal(R[q].reshape(NQ, NQ, H, N0c), S[q * N0c:(q + 1) * N0c].transpose(3, 2, 1, 0))
    O = []
    for q in range(world):
        view = R[q].reshape(NQ, NQ, H, N0c)
        o = np.empty(world * blk, dtype=complex)
        for r in range(world):
            o[r * blk:(r + 1) * blk] = view[r * slab:(r + 1) * slab].transpose(3, 2, 0, 1).reshape(-1)
        O.append(o)
    T = [np.full(world * blk, np.nan + 0j) for _ in range(world)]
    for i in range(C2):
        kb, ke = N0c * i // C2, N0c * (i + 1) // C2
        partial = []
        for q in range(world):                     # K2 has written k0 (local) < ke only
            o = np.full(world * blk, np.nan + 0j)
            for r in range(world):
                lo = r * blk
                o[lo:lo + ke * inner2] = O[q][lo:lo + ke * inner2]
            partial.append(o)
        pc = _chunk(world, blk, 1, inner2, kb, ke)
        for src, dst, so, do, nb in pc:
            assert np.isnan(T[dst][do // 16:(do + nb) // 16].real).all()
        _apply(pc, partial, T)
    for r in range(world):
        assert np.array_equal(T[r].reshape(N, H, slab, NQ), S[:, :, :, r * slab:(r + 1) * slab].transpose(0, 1, 3, 2))

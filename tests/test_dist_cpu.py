"""The N>1 host logic on CPU: world_size-2 gloo process group (127.0.0.1)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2412_07240_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r, w, lr = D.env()
    t = D.max_over_ranks(1.5 + rank)          # per-rank "time"
    # the sharded filter's NCCL id travels from rank 0 exactly as bench.py sends it
    obj = [bytes(range(128)) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    dist.barrier()
    q.put((r, w, lr, t, D.rank_seed(5, r), D.shard(4096, r, w), obj[0]))
    dist.destroy_process_group()


def test_gloo_world2_max_over_ranks_and_sharding():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    out = sorted(q.get(timeout=10) for _ in range(2))
    assert [o[0] for o in out] == [0, 1] and all(o[1] == 2 for o in out)
    assert all(o[3] == 2.5 for o in out)                 # max over ranks, seen by every rank
    assert out[0][4] != out[1][4]                         # distinct per-rank seeds (weak scaling)
    assert out[0][5] == (0, 2048) and out[1][5] == (2048, 4096)
    assert out[0][6] == out[1][6] == bytes(range(128))      # id broadcast for pmf_create_sharded


def test_create_sharded_validates_before_touching_a_gpu():
    """pmf_create_sharded argument checks run on the host (CPU box): slab divisibility,
    batch, nx; a real (non-virtual) create without a device fails loudly."""
    import ctypes as C
    import numpy as np
    from paper_2412_07240_b200 import pmf
    lib = pmf.load_library()
    cfg = pmf.pmf_config()
    cfg.nx, cfg.batch = 4, 1
    for i, v in enumerate((8, 6, 12, 8)):
        cfg.n[i] = v
    A = np.zeros(16)
    Q = np.eye(4).reshape(-1)
    h = C.c_void_p()
    uid = C.create_string_buffer(128)
    rc = lib.pmf_create_sharded(C.byref(cfg), pmf._dptr(A), pmf._dptr(Q), 0, 3, uid, C.byref(h))
    assert rc == -1                                   # 8 planes cannot split into 3 slabs
    cfg.batch = 2
    rc = lib.pmf_create_sharded(C.byref(cfg), pmf._dptr(A), pmf._dptr(Q), 0, 2, uid, C.byref(h))
    assert rc == -1                                   # one filter per sharded context
    cfg.batch = 1
    rc = lib.pmf_create_sharded(C.byref(cfg), pmf._dptr(A), pmf._dptr(Q), 5, 2, uid, C.byref(h))
    assert rc == -1                                   # rank out of range


@pytest.mark.parametrize("batch,world", [(4096, 8), (7, 3), (1, 2)])
def test_shard_partition(batch, world):
    ranges = [D.shard(batch, r, world) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == batch
    for (a, b), (c, d) in zip(ranges, ranges[1:]):
        assert b == c and b >= a
    assert max(b - a for a, b in ranges) - min(b - a for a, b in ranges) <= 1

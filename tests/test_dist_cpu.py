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
    dist.barrier()
    q.put((r, w, lr, t, D.rank_seed(5, r), D.shard(4096, r, w)))
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


@pytest.mark.parametrize("batch,world", [(4096, 8), (7, 3), (1, 2)])
def test_shard_partition(batch, world):
    ranges = [D.shard(batch, r, world) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == batch
    for (a, b), (c, d) in zip(ranges, ranges[1:]):
        assert b == c and b >= a
    assert max(b - a for a, b in ranges) - min(b - a for a, b in ranges) <= 1

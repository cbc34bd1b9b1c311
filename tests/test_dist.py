"""The N>1 plumbing of bench.py on CPU: gloo, world size 2, 127.0.0.1."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2211_03715_b200 import dist as tdist


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    r, w = tdist.init("gloo")
    assert (r, w) == (rank, world)
    tdist.barrier()
    mx = tdist.max_over_ranks(10.0 + 5.0 * rank)        # rank 1 is the slow one
    total = tdist.sum_over_ranks(32.0)                   # images processed, weak scaling
    out.put((rank, mx, total))
    tdist.finalize()


def test_gloo_world2_max_and_sum_over_ranks():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[0] for r in res] == [0, 1]
    assert all(r[1] == 15.0 for r in res)      # every rank sees the max
    assert all(r[2] == 64.0 for r in res)


@pytest.mark.parametrize("B,world", [(64, 8), (64, 3), (7, 4), (1, 2), (0, 2)])
def test_shard_covers_batch_exactly(B, world):
    seen = []
    for r in range(world):
        start, n = tdist.shard(B, world, r)
        seen.extend(range(start, start + n))
    assert seen == list(range(B))
    sizes = [tdist.shard(B, world, r)[1] for r in range(world)]
    assert max(sizes) - min(sizes) <= 1


def test_single_process_is_identity():
    assert tdist.max_over_ranks(3.5) == 3.5
    assert tdist.sum_over_ranks(2.0) == 2.0
    with pytest.raises(ValueError):
        tdist.shard(4, 0, 0)

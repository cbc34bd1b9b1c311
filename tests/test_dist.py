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


def _shard_worker(rank, world, port, global_batch, out):
    """Batch-sharded inference on CPU (the oracle model stands in for the GPU forward):
    this rank evaluates its shard of the global batch, the logits are all-gathered in
    global-batch order and compared with the unsharded evaluation by the caller."""
    import torch

    import oracle.model as om
    import synth.models as sm
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    tdist.init("gloo")
    sh = tdist.BatchShard(global_batch)
    ops = sm.tucker_resnet(18, image=16, num_classes=10, width=8, seed=5)   # identical on every rank
    x = sm.model_input(sh.count, image=16, seed=3, first=sh.start)         # this rank's images
    local = torch.from_numpy(om.forward(ops, x).reshape(sh.count, -1))
    full = sh.gather(local)
    out.put((rank, sh.start, sh.count, full.numpy(), local.numpy()))
    tdist.finalize()


@pytest.mark.parametrize("global_batch", [4, 3])
def test_gloo_world2_sharded_forward_gather_equals_unsharded(global_batch):
    import numpy as np

    import oracle.model as om
    import synth.models as sm
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, global_batch, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [(r[1], r[2]) for r in res] == [tdist.shard(global_batch, world, r) for r in range(world)]
    ops = sm.tucker_resnet(18, image=16, num_classes=10, width=8, seed=5)
    ref = om.forward(ops, sm.model_input(global_batch, image=16, seed=3)).reshape(global_batch, -1)
    for r in res:
        # the gather is exact: every rank holds every rank's rows, in global-batch order
        for q in res:
            assert np.array_equal(r[3][q[1]:q[1] + q[2]], q[4])
        # and the sharded result is the unsharded one (fp64; the FC's BLAS matmul may block
        # differently for a different batch size, so equality is to rounding, not bits)
        assert r[3].shape == ref.shape
        assert np.max(np.abs(r[3] - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_model_input_shards_are_slices_of_the_global_batch():
    import numpy as np

    import synth
    import synth.models as sm
    full = sm.model_input(5, image=8, seed=1)
    assert np.array_equal(sm.model_input(2, image=8, seed=1, first=3), full[3:])
    s = synth.LayerShape(6, 4, 4, 5, 5, 2, 2)
    xs = synth.make_images(s, 0, 6, layer_id=2)
    assert np.array_equal(synth.make_images(s, 4, 2, layer_id=2), xs[4:])

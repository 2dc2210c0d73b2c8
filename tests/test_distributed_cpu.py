"""World-size-2 gloo tests of the multi-GPU host logic (no GPU needed).

Checks that example sharding partitions the batch, that transforms drawn
for the whole batch and sliced per rank equal the single-process draw, and
that the optional gradient gather reassembles rows in rank order.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        from pathlib import Path

        sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
        from paper_1912_04822_b200 import distributed as D
        from paper_1912_04822_b200 import geom

        n = 11
        centers = np.random.default_rng(0).uniform(-2, 2, (n, 3))
        full = geom.draw_transform_array(centers, 2.0, True, np.random.default_rng(9))
        mine = D.shard_transforms(full, rank, world)
        start, stop = D.shard_range(n, rank, world)
        local = torch.arange(start * 3, stop * 3, dtype=torch.float32).reshape(-1, 3)
        gathered = D.gather_rows(local)
        slowest = D.max_over_ranks(float(rank + 1))
        q.put((rank, start, stop, mine.packed.tolist(), gathered.numpy().tolist(), slowest))
    finally:
        dist.destroy_process_group()


def test_world2_sharding_and_gather():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_1912_04822_b200 import geom

    n = 11
    centers = np.random.default_rng(0).uniform(-2, 2, (n, 3))
    full = geom.draw_transform_array(centers, 2.0, True, np.random.default_rng(9)).packed
    covered = []
    for rank, start, stop, mine, gathered, slowest in results:
        covered.extend(range(start, stop))
        np.testing.assert_array_equal(np.array(mine), full[start:stop])
        np.testing.assert_array_equal(np.array(gathered),
                                      np.arange(n * 3, dtype=np.float32).reshape(n, 3))
        assert slowest == 2.0
    assert covered == list(range(n))


def test_shard_range_partitions():
    from paper_1912_04822_b200.distributed import shard_range

    for n in (0, 1, 7, 50, 400):
        for w in (1, 2, 3, 8):
            parts = [shard_range(n, r, w) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)

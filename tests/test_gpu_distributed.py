"""The multi-GPU path on the GPU box (which exposes one B200):

* two ranks (gloo for the host collectives, both gridding on cuda:0): each
  grids its contiguous shard of a global batch with the transforms drawn for
  the whole batch and sliced; the gathered coordinate
  gradients and the shards' grids equal the single-process run bit for bit;
* one rank over NCCL: ``gather_rows`` / ``max_over_ranks`` on CUDA tensors
  run through NCCL (the collective the optional gather uses on 8 GPUs).
"""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _batch():
    from paper_1912_04822_b200 import synthetic

    exs = synthetic.batch(7, seed=2)
    centers = np.stack([ex.coord_sets[-1].centroid() for ex in exs])
    return exs, centers


def _grid_shard(exs, centers, rank, world):
    from paper_1912_04822_b200 import GridMaker, distributed, geom

    full = geom.draw_transform_array(centers, 2.0, True, np.random.default_rng(11))
    mine = distributed.shard_transforms(full, rank, world)
    sub = distributed.shard(exs, rank, world)
    gm = GridMaker(device="cuda:0")
    pb = gm.pack(sub)
    out, _ = gm.forward_packed(pb, transforms=mine)
    cg, _ = gm.backward_packed(pb, out, reuse_prepared=True)  # gradient of 1/2 |grid|^2
    return out, cg


def _worker(rank, world, port, backend, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    torch.cuda.set_device(0)
    kw = {"device_id": torch.device("cuda", 0)} if backend == "nccl" else {}
    dist.init_process_group(backend, rank=rank, world_size=world, **kw)
    try:
        from paper_1912_04822_b200 import distributed

        exs, centers = _batch()
        out, cg = _grid_shard(exs, centers, rank, world)
        torch.cuda.synchronize()
        if backend == "nccl":
            allg = distributed.gather_rows(cg)                 # NCCL all-gather on CUDA
            slow = distributed.max_over_ranks(float(rank) + 0.5, device="cuda:0")
        else:
            allg = distributed.gather_rows(cg.cpu())           # gloo on host copies
            slow = distributed.max_over_ranks(float(rank) + 0.5)
        q.put((rank, out.cpu().numpy(), allg.cpu().numpy(), slow))
    finally:
        dist.destroy_process_group()


def _run(world, backend):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, backend, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return sorted(res, key=lambda r: r[0])


def _single():
    exs, centers = _batch()
    out, cg = _grid_shard(exs, centers, 0, 1)
    return out.cpu().numpy(), cg.cpu().numpy()


def test_two_ranks_shard_and_gather_bit_identical():
    out1, cg1 = _single()
    res = _run(2, "gloo")
    np.testing.assert_array_equal(np.concatenate([r[1] for r in res]), out1)
    for _, _, allg, slow in res:
        np.testing.assert_array_equal(allg, cg1)
        assert slow == 1.5


def test_nccl_gather_on_cuda_tensors():
    out1, cg1 = _single()
    (rank, out, allg, slow), = _run(1, "nccl")
    np.testing.assert_array_equal(out, out1)
    np.testing.assert_array_equal(allg, cg1)
    assert slow == 0.5

"""GPU parity at exactly the inputs ``bench.py`` grids (configs C1-C5).

Each test builds the bench's own batch (``bench.make_batch``: same seeds,
same 50 examples per GPU, C1's single ligand), draws the transforms the way
the bench step does (``geom.draw_transform_array`` over the batch's default
centers: random rotation + 2 A translation), runs the bench's API path
(``pack`` -> ``forward_packed`` -> ``backward_packed(reuse_prepared=True)``
with a seeded N(0,1) ``grid_grad`` on the device) and compares every output
with the CPU oracle on the same inputs (the oracle draws the same transforms
from the same seed; tests/test_cpu_host.py pins the draw equivalence).

C5 (96^3) is compared example by example (50 grids are 4.95 GB); the device
run is the full 50-example launch the bench times.
"""

import numpy as np
import pytest

import oracle
from parity import assert_close

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _bench():
    import bench

    return bench


def _run_bench_path(cfg, rti=False, seed=1234):
    """The bench step on this config; returns what the oracle comparison needs."""
    from paper_1912_04822_b200 import GridMaker, geom

    b = _bench()
    exs, centers = b.make_batch(cfg, 0, 1)
    dev = torch.device("cuda", 0)
    gm = GridMaker(resolution=cfg["resolution"], dimension=cfg["dimension"],
                   binary=cfg["binary"], radius_type_indexed=rti, device=dev)
    D = gm.points_per_side()
    pb = gm.pack(exs)
    N, C = pb.nexamples, pb.nchannels
    out = torch.empty((N, C, D, D, D), dtype=torch.float32, device=dev)
    gg = torch.randn((N, C, D, D, D), generator=torch.Generator(device=dev).manual_seed(7),
                     device=dev, dtype=torch.float32)
    xf = geom.draw_transform_array(centers, 2.0, True, np.random.default_rng(seed))
    gm.forward_packed(pb, out, transforms=xf)
    cg, tg = gm.backward_packed(pb, gg, reuse_prepared=True)
    torch.cuda.synchronize(dev)
    go = oracle.GridOracle(resolution=cfg["resolution"], dimension=cfg["dimension"],
                           binary=cfg["binary"], radius_type_indexed=rti)
    _, ocenters, origins, placed, _ = go.place(exs, random_rotation=True, random_translation=2.0,
                                              rng=np.random.default_rng(seed))
    return gm, pb, exs, out, gg, cg, tg, go, ocenters, origins, placed


def _oracle_forward(go, placed, origins, e0, e1, C, D):
    sub = [(e - e0, choff, cs, c64) for (e, choff, cs, c64) in placed if e0 <= e < e1]
    ref = np.zeros((e1 - e0, C, D, D, D), np.float32)
    go.forward_placed(ref, sub, origins[e0:e1])
    return ref


def _check(cfg_name, rti=False, chunk=50):
    b = _bench()
    cfg = b.CONFIGS[cfg_name]
    gm, pb, exs, out, gg, cg, tg, go, ocenters, origins, placed = _run_bench_path(cfg, rti)
    N, C = pb.nexamples, pb.nchannels
    D = gm.points_per_side()
    assert N == cfg["batch"]
    cg = cg.cpu().numpy()
    tg = tg.cpu().numpy() if tg is not None else None
    for e0 in range(0, N, chunk):
        e1 = min(N, e0 + chunk)
        got = out[e0:e1].cpu().numpy()
        ref = _oracle_forward(go, placed, origins, e0, e1, C, D)
        if cfg["binary"]:
            np.testing.assert_array_equal(got, ref, err_msg=f"{cfg_name} binary [{e0},{e1})")
        else:
            assert_close(got, ref, what=f"{cfg_name} forward [{e0},{e1})")
    # backward: the reference's per-(example, set) loop in the forward's frame
    ggh = None
    for (e, choff, cs, a0, w0) in pb.placed:
        if ggh is None or ggh[0] != e:
            ggh = (e, gg[e].cpu().numpy())
        c64 = next(c for (pe, pch, pcs, c) in placed if pe == e and pch == choff)
        ocg, otg = go.backward(cs, ggh[1][choff:choff + cs.num_types], center=ocenters[e],
                               coords64=c64)
        na = cs.coords.shape[0]
        assert_close(cg[a0:a0 + na], ocg, what=f"{cfg_name} coord grad e{e} set@{choff}")
        if pb.vector_mode:
            assert_close(tg[w0:w0 + na * cs.num_types].reshape(na, cs.num_types), otg,
                         what=f"{cfg_name} type grad e{e} set@{choff}")


def test_c1_bench_config():
    """C1: one 30-atom ligand (seed 1), 14 channels, batch 1."""
    _check("c1")


def test_c2_bench_config():
    _check("c2")


def test_c3_bench_config_binary_bit_exact():
    _check("c3")


@pytest.mark.parametrize("rti", [False, True])
def test_c4_bench_config_full_batch(rti):
    """C4: the full 50-example vector-typed batch, coordinate and type grads."""
    _check("c4", rti=rti)


def test_c5_bench_config_full_batch():
    """C5: 96^3, the full 50-example per-GPU batch, compared 5 grids at a time."""
    _check("c5", chunk=5)

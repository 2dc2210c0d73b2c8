"""GPU regression tests for round-2 fixes, each against the CPU oracle:

* index-mode ``grid_atoms`` with coordinates that differ from the packed
  ones (the prepare pass reads per-slot records gathered at pack time; they
  must follow ``load_coords``);
* ``backward_packed(reuse_prepared=False)`` queued right behind other work
  (the backward follows its own prepare pass, which triggers dependents
  before its stores: the backward must not read its records early);
* the exact-transform fallback when numpy's matmul rounding cannot be
  calibrated (host-transformed f64 positions, binary stays bit-exact);
* Grid views (``grids.py``) as ``out`` / ``grid_grad``.
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


def _perturbed(exs, rng, scale=0.37):
    from paper_1912_04822_b200 import Example

    out = []
    for ex in exs:
        sets = [cs.with_coords((cs.coords + rng.normal(0, scale, cs.coords.shape))
                               .astype(np.float32)) for cs in ex.coord_sets]
        out.append(Example(coord_sets=sets))
    return out


def test_grid_atoms_index_mode_with_new_coordinates():
    from paper_1912_04822_b200 import GridMaker, geom, synthetic
    from paper_1912_04822_b200.autograd import grid_atoms

    exs = synthetic.batch(5, seed=21)
    moved = _perturbed(exs, np.random.default_rng(4))
    gm = GridMaker()
    pb = gm.pack(exs)  # packed with the ORIGINAL coordinates
    xf = geom.draw_transform_array(pb.default_centers, 2.0, True, np.random.default_rng(9))
    x = torch.from_numpy(np.concatenate([cs.coords for ex in moved for cs in ex.coord_sets])) \
        .cuda().requires_grad_(True)
    grid = grid_atoms(gm, pb, x, transforms=xf)
    G = torch.randn(grid.shape, generator=torch.Generator(device="cuda").manual_seed(5),
                    device="cuda")
    (grid * G).sum().backward()
    go = oracle.GridOracle()
    # same centers as the batch (pack-time defaults of the original coordinates)
    ref = go.forward_batch(moved, centers=pb.default_centers, random_rotation=True,
                           random_translation=2.0, rng=np.random.default_rng(9))
    assert_close(grid.detach().cpu().numpy(), ref, what="forward with new coordinates")
    cgs, _ = go.backward_batch(moved, G.cpu().numpy(), centers=pb.default_centers,
                               random_rotation=True, random_translation=2.0,
                               rng=np.random.default_rng(9))
    want = np.concatenate([np.asarray(cg, np.float64) @ xf.packed[e, :9].reshape(3, 3)
                           for cg, (e, _, _, _, _) in zip(cgs, pb.placed)])
    assert_close(x.grad.cpu().numpy(), want, what="dL/dx with new coordinates")


def test_backward_after_its_own_prepare_queued():
    """Several backward_packed(reuse_prepared=False) calls queued without a
    host sync, each behind a forward of ANOTHER transform of the same batch."""
    from paper_1912_04822_b200 import GridMaker, geom, synthetic

    exs = synthetic.batch(12, seed=2)
    gm = GridMaker()
    pb = gm.pack(exs)
    gg = torch.randn((12, 28, 48, 48, 48), generator=torch.Generator(device="cuda").manual_seed(1),
                     device="cuda")
    out = torch.empty_like(gg)
    xfs = [geom.draw_transform_array(pb.default_centers, 2.0, True, np.random.default_rng(s))
           for s in range(4)]
    results = []
    for k in range(4):
        gm.forward_packed(pb, out, transforms=xfs[(k + 1) % 4])  # a different frame
        cg, _ = gm.backward_packed(pb, gg, transforms=xfs[k])   # prepare + backward
        results.append(cg.clone())
    torch.cuda.synchronize()
    go = oracle.GridOracle()
    ggh = gg.cpu().numpy()
    for k in range(4):
        cgs, _ = go.backward_batch(exs, ggh, random_rotation=True, random_translation=2.0,
                                   rng=np.random.default_rng(k))
        assert_close(results[k].cpu().numpy(), np.concatenate(cgs), what=f"backward {k}")


def test_exact_transform_fallback_bit_exact(monkeypatch, rng):
    from conftest import random_coordinate_set
    from paper_1912_04822_b200 import Example, GridMaker, geom, synthetic

    monkeypatch.setattr(geom, "_ORDER_CACHE", {1: -1, 2: -1})
    exs = synthetic.batch(8, seed=2)
    exs += [Example(coord_sets=[random_coordinate_set(rng, 1, 14, 4.0),
                                random_coordinate_set(rng, 2, 14, 4.0)]) for _ in range(8)]
    gm = GridMaker(binary=True)
    with pytest.warns(RuntimeWarning, match="transformed on the host"):
        import paper_1912_04822_b200.voxelizer as vz

        monkeypatch.setattr(vz, "_FALLBACK_WARNED", [False])
        grid = gm.forward_batch(exs, random_rotation=True, random_translation=2.0,
                                rng=np.random.default_rng(0))
    ref = oracle.GridOracle(binary=True).forward_batch(
        exs, random_rotation=True, random_translation=2.0, rng=np.random.default_rng(0))
    np.testing.assert_array_equal(grid, ref)
    # smooth mode and the backward take the same host positions
    gs = GridMaker()
    g2, xf = gs.forward_batch(exs[:8], random_rotation=True, random_translation=2.0,
                              rng=np.random.default_rng(3), return_transforms=True)
    go = oracle.GridOracle()
    r2 = go.forward_batch(exs[:8], random_rotation=True, random_translation=2.0,
                          rng=np.random.default_rng(3))
    assert_close(g2, r2, what="fallback smooth forward")
    res = gs.backward_batch(exs[:8], r2, transforms=xf)
    cgs, _ = go.backward_batch(exs[:8], r2, random_rotation=True, random_translation=2.0,
                               rng=np.random.default_rng(3))
    assert_close(np.concatenate([c for ex in res for (c, _) in ex]), np.concatenate(cgs),
                 what="fallback backward")


def test_grid_views_as_out_and_grid_grad(rng):
    from conftest import random_coordinate_set
    from paper_1912_04822_b200 import GridMaker, make_grid, view_over

    cs = random_coordinate_set(rng, 25, 4, 5.0)
    gm = GridMaker(dimension=10.0)
    D = gm.points_per_side()
    go = oracle.GridOracle(dimension=10.0)
    ref = go.forward(cs)
    # host view over a flat numpy buffer
    buf = np.full(4 * D ** 3, 7.0, np.float32)
    hv = view_over(buf, (4, D, D, D), "f32")
    res = gm.forward(cs, out=hv)
    assert res is hv.array
    assert_close(buf.reshape(4, D, D, D), ref, what="numpy-backed view")
    # device grid: make_grid(device=...) and a view over a CUDA tensor
    dg = make_grid((4, D, D, D), device="cuda")
    assert dg.on_device
    res = gm.forward(cs, out=dg)
    assert res is dg.array
    assert_close(dg.tonumpy(), ref, what="device grid")
    t = torch.zeros(4 * D ** 3 + 5, device="cuda")
    tv = view_over(t, (4, D, D, D))
    gm.forward(cs, out=tv)
    assert_close(t[:4 * D ** 3].view(4, D, D, D).cpu().numpy(), ref, what="tensor view")
    # grid_grad as views (host and device) -> same gradients as the oracle
    gg = rng.standard_normal((4, D, D, D)).astype(np.float32)
    want, _ = go.backward(cs, gg)
    cg_h, _ = gm.backward(cs, view_over(gg, (4, D, D, D)))
    assert_close(cg_h, want, what="grad via host view")
    cg_d, _ = gm.backward(cs, view_over(torch.from_numpy(gg).cuda(), (4, D, D, D)))
    assert_close(cg_d.cpu().numpy(), want, what="grad via device view")

    class Duck:  # any object with .array (the reference's own GridView is one)
        def __init__(self, a):
            self.array = a

    out = np.zeros((1, 4, D, D, D), np.float32)
    gm.forward_batch([cs], out=Duck(out))
    assert_close(out[0], ref, what="duck-typed grid")


def test_numpy_api_pack_cache_hits_and_invalidates(monkeypatch):
    """forward_batch -> backward_batch on the same examples packs once; an
    in-place coordinate change (same objects) repacks."""
    import paper_1912_04822_b200.voxelizer as vz
    from paper_1912_04822_b200 import GridMaker, synthetic

    exs = synthetic.batch(3, seed=2)
    gm = GridMaker()
    calls = []
    real = vz.PackedBatch

    def counting(*a, **k):
        calls.append(1)
        return real(*a, **k)

    monkeypatch.setattr(vz, "PackedBatch", counting)
    g1, xf = gm.forward_batch(exs, random_rotation=True, random_translation=2.0,
                              rng=np.random.default_rng(0), return_transforms=True)
    res = gm.backward_batch(exs, g1, transforms=xf)
    assert len(calls) == 1
    go = oracle.GridOracle()
    cgs, _ = go.backward_batch(exs, g1, random_rotation=True, random_translation=2.0,
                               rng=np.random.default_rng(0))
    assert_close(np.concatenate([c for ex in res for (c, _) in ex]), np.concatenate(cgs),
                 what="cached-pack backward")
    exs[1].coord_sets[0].coords[5] += np.float32(0.75)  # in place: same objects
    g2 = gm.forward_batch(exs)
    assert len(calls) == 2
    assert_close(g2, go.forward_batch(exs), what="repacked after an in-place change")


def test_numpy_api_concurrent_threads_and_pickling():
    """Threads sharing one GridMaker and the same examples each get their own
    packed batch (the pack cache is per thread), so concurrent forward_batch
    calls with different augmentation equal the sequential ones; a used
    GridMaker still pickles / deep-copies as its parameters."""
    import copy
    import pickle
    import threading

    from paper_1912_04822_b200 import GridMaker, synthetic

    exs = synthetic.batch(6, seed=3)
    gm = GridMaker()
    want = [gm.forward_batch(exs, random_rotation=True, random_translation=2.0,
                             rng=np.random.default_rng(s)) for s in range(4)]
    got = [None] * 4
    barrier = threading.Barrier(4)

    def work(s):
        torch.cuda.set_device(0)
        with torch.cuda.stream(torch.cuda.Stream()):
            barrier.wait()
            for _ in range(3):
                got[s] = gm.forward_batch(exs, random_rotation=True, random_translation=2.0,
                                          rng=np.random.default_rng(s))

    ts = [threading.Thread(target=work, args=(s,)) for s in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for s in range(4):
        np.testing.assert_array_equal(got[s], want[s])
    for clone in (pickle.loads(pickle.dumps(gm)), copy.deepcopy(gm)):
        assert clone.get_params() == gm.get_params()
        np.testing.assert_array_equal(clone.forward_batch(exs[:2]), gm.forward_batch(exs[:2]))

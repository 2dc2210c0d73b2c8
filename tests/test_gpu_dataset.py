"""Device-side batch assembly (dataset.py, csrc/assemble.cu): a batch built
on the GPU from a resident dataset equals the host packing of the same
examples array for array (except the backward launch order), its forward job
table equals the host builder's entry for entry, and its grids / gradients
equal both the host-packed path (bit for bit) and the CPU oracle."""

import ctypes

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


@pytest.fixture(scope="module")
def data():
    from conftest import random_coordinate_set
    from paper_1912_04822_b200 import Example, synthetic
    from paper_1912_04822_b200.dataset import DeviceDataset

    exs = synthetic.batch(40, seed=2)
    rng = np.random.default_rng(5)
    # odd shapes: a single-atom set, an empty set, a far-away atom
    for k in range(6):
        sets = [random_coordinate_set(rng, [1, 0, 7, 30, 2, 13][k], 14, 9.0),
                random_coordinate_set(rng, [5, 9, 0, 1, 40, 3][k], 14, 4.0)]
        exs.append(Example(coord_sets=sets))
    return exs, DeviceDataset(exs)


def _host_array(pb, name, n):
    off, dt, shape = pb.offsets[name]
    return np.frombuffer(pb.host.numpy()[off:off + n * np.dtype(dt).itemsize].tobytes(), dt)


def _dev_array(ab, name, n):
    off, dt, shape = ab.offsets[name]
    return ab.dev[off:off + n * np.dtype(dt).itemsize].cpu().numpy().view(dt)


@pytest.mark.parametrize("seed,cfg", [(0, dict()), (1, dict()),
                                      (2, dict(resolution=0.25, dimension=23.75)),
                                      (3, dict(resolution=0.375, dimension=11.3, radius_scale=0.8))])
def test_assembled_batch_equals_host_packing(data, seed, cfg):
    from paper_1912_04822_b200 import GridMaker, _native

    exs, ds = data
    gm = GridMaker(**cfg)
    ids = np.random.default_rng(seed).permutation(len(exs))[:37]
    ab = ds.batch(50).assemble(gm, ids)
    pb = gm.pack([exs[i] for i in ids])
    torch.cuda.synchronize()
    assert (ab.nexamples, ab.natoms, ab.nsets, ab.nsegs, ab.max_seg_items,
            ab.max_example_items) == (pb.nexamples, pb.natoms, pb.nsets, pb.nsegs,
                                       pb.max_seg_items, pb.max_example_items)
    A, S, N, C = pb.natoms, pb.nsets, pb.nexamples, pb.nchannels
    for name, n in (("coords32", 3 * A), ("atom_radius", A), ("atom_set", A), ("atom_type", A),
                    ("set_start", S), ("set_end", S), ("set_example", S), ("set_choff", S),
                    ("set_t", S), ("ex_item_start", N), ("ex_item_end", N), ("item_perm", A),
                    ("chan_off", N * (C + 1)), ("segs", pb.nsegs)):
        np.testing.assert_array_equal(_dev_array(ab, name, n), _host_array(pb, name, n),
                                      err_msg=name)
    from paper_1912_04822_b200.packing import _SLOT_DTYPE

    got = _dev_array(ab, "slot_rec", 48 * A).view(_SLOT_DTYPE)
    want = _host_array(pb, "slot_rec", 48 * A).view(_SLOT_DTYPE)
    for f in ("x", "y", "z", "atom", "ch", "ex", "single", "r"):
        np.testing.assert_array_equal(got[f], want[f], err_msg=f"slot_rec.{f}")
    # backward launch order: a permutation (per example here)
    bs = _dev_array(ab, "bwd_slot", A)
    assert np.array_equal(np.sort(bs), np.arange(A))
    # forward job table == the host builder's
    p = gm._gm_params(gm.points_per_side())
    co = np.ascontiguousarray(_host_array(pb, "chan_off", N * (C + 1)))
    L = _native.lib()
    cnt = L.gm_forward_jobs(ctypes.byref(p), N, C, co.ctypes.data, None, 0)
    jobs = np.zeros((cnt, 4), np.int32)
    L.gm_forward_jobs(ctypes.byref(p), N, C, co.ctypes.data, jobs.ctypes.data, cnt)
    assert ab._gm.nfwd_jobs == cnt
    np.testing.assert_array_equal(ab._jobs[:cnt].cpu().numpy(), jobs)


@pytest.mark.parametrize("cfg", [dict(), dict(binary=True), dict(resolution=0.25, dimension=23.75),
                                 dict(resolution=0.375, dimension=11.3),
                                 dict(resolution=0.25, dimension=6.0, radius_scale=1.3)])
def test_assembled_forward_backward_bitwise_and_vs_oracle(data, cfg):
    from paper_1912_04822_b200 import GridMaker, geom

    exs, ds = data
    gm = GridMaker(**cfg)
    D = gm.points_per_side()
    ab = ds.batch(12)
    rng = np.random.default_rng(3)
    for step in range(3):  # the same batch object, re-assembled each step
        ids = rng.permutation(len(exs))[:12 if D < 90 else 3]
        ab.assemble(gm, ids)
        sub = [exs[i] for i in ids]
        xf = geom.draw_transform_array(ab.default_centers, 2.0, True, np.random.default_rng(step))
        out = torch.empty((len(ids), 28, D, D, D), device="cuda")
        gm.forward_packed(ab, out, transforms=xf)
        gg = torch.randn_like(out)
        cg, _ = gm.backward_packed(ab, gg, reuse_prepared=True)
        pb = gm.pack(sub)
        out2 = torch.empty_like(out)
        gm.forward_packed(pb, out2, transforms=xf)
        cg2, _ = gm.backward_packed(pb, gg, reuse_prepared=True)
        assert torch.equal(out, out2), f"step {step}: grids differ from the host-packed batch"
        assert torch.equal(cg, cg2), f"step {step}: gradients differ from the host-packed batch"
    go = oracle.GridOracle(**cfg)
    ref = go.forward_batch(sub, random_rotation=True, random_translation=2.0,
                           rng=np.random.default_rng(2))
    if gm.binary:
        np.testing.assert_array_equal(out.cpu().numpy(), ref)
    else:
        assert_close(out.cpu().numpy(), ref, what="assembled forward vs oracle")
        cgs, _ = go.backward_batch(sub, gg.cpu().numpy(), random_rotation=True,
                                   random_translation=2.0, rng=np.random.default_rng(2))
        assert_close(cg.cpu().numpy(), np.concatenate(cgs), what="assembled backward vs oracle")


@pytest.fixture(scope="module")
def vdata():
    from conftest import random_coordinate_set
    from paper_1912_04822_b200 import Example, make_vector_types, synthetic
    from paper_1912_04822_b200.dataset import DeviceDataset

    exs = synthetic.batch(16, seed=4, vector=True)
    rng = np.random.default_rng(6)
    for k in range(4):  # odd shapes: single-atom and empty sets
        a = make_vector_types(random_coordinate_set(rng, [1, 0, 9, 25][k], 14, 8.0))
        b = make_vector_types(random_coordinate_set(rng, [7, 3, 0, 1][k], 14, 4.0))
        exs.append(Example(coord_sets=[a, b]))
    return exs, DeviceDataset(exs)


@pytest.mark.parametrize("rti", [False, True])
def test_vector_assembled_batch_equals_host_packing(vdata, rti):
    from paper_1912_04822_b200 import GridMaker

    exs, ds = vdata
    gm = GridMaker(radius_type_indexed=rti)
    # the odd examples (index >= 16) carry no type radii: type-indexed radii
    # take the synthetic ones only, as the host packing requires
    ids = np.random.default_rng(3).permutation(16 if rti else len(exs))[:13]
    ab = ds.batch(16).assemble(gm, ids)
    pb = gm.pack([exs[i] for i in ids])
    torch.cuda.synchronize()
    assert (ab.nexamples, ab.natoms, ab.nitems, ab.nsets, ab.nsegs, ab.max_seg_items,
            ab.max_example_items, ab.nweights) == (pb.nexamples, pb.natoms, pb.nitems, pb.nsets,
                                                   pb.nsegs, pb.max_seg_items,
                                                   pb.max_example_items, pb.nweights)
    A, S, N, C, I = pb.natoms, pb.nsets, pb.nexamples, pb.nchannels, pb.nitems
    for name, n in (("coords32", 3 * A), ("atom_radius", A), ("atom_set", A),
                    ("set_start", S), ("set_end", S), ("set_example", S), ("set_choff", S),
                    ("set_t", S), ("set_wstart", S), ("set_trstart", S),
                    ("weights", pb.nweights), ("type_radius", pb.offsets["type_radius"][2][0]),
                    ("item_atom", I), ("item_channel", I), ("item_weight", I),
                    ("item_radius", I), ("ex_item_start", N), ("ex_item_end", N),
                    ("item_perm", I), ("chan_off", N * (C + 1)), ("segs", pb.nsegs),
                    ("bwd_slot", A)):
        np.testing.assert_array_equal(_dev_array(ab, name, n), _host_array(pb, name, n),
                                      err_msg=name)


@pytest.mark.parametrize("rti", [False, True])
def test_vector_assembled_forward_backward(vdata, rti):
    from paper_1912_04822_b200 import GridMaker, geom

    exs, ds = vdata
    gm = GridMaker(radius_type_indexed=rti)
    ab = ds.batch(8)
    ids = np.random.default_rng(8).permutation(16 if rti else len(exs))[:8]
    ab.assemble(gm, ids)
    sub = [exs[i] for i in ids]
    xf = geom.draw_transform_array(ab.default_centers, 2.0, True, np.random.default_rng(4))
    out, _ = gm.forward_packed(ab, transforms=xf)
    gg = torch.randn_like(out)
    cg, tg = gm.backward_packed(ab, gg, reuse_prepared=True)
    pb = gm.pack(sub)
    out2, _ = gm.forward_packed(pb, transforms=xf)
    cg2, tg2 = gm.backward_packed(pb, gg, reuse_prepared=True)
    assert torch.equal(out, out2)
    assert torch.equal(cg, cg2) and torch.equal(tg, tg2)
    go = oracle.GridOracle(radius_type_indexed=rti)
    ref = go.forward_batch(sub, random_rotation=True, random_translation=2.0,
                           rng=np.random.default_rng(4))
    assert_close(out.cpu().numpy(), ref, what="vector assembled forward vs oracle")
    cgs, tgs = go.backward_batch(sub, gg.cpu().numpy(), random_rotation=True,
                                 random_translation=2.0, rng=np.random.default_rng(4))
    assert_close(cg.cpu().numpy(), np.concatenate(cgs), what="coord grads")
    assert_close(tg.cpu().numpy(), np.concatenate([t.reshape(-1) for t in tgs]),
                 what="type grads")


def test_vector_type_radii_required_when_type_indexed(vdata):
    from paper_1912_04822_b200 import ConfigError, GridMaker

    exs, ds = vdata
    with pytest.raises(ConfigError, match="type_radii is missing"):
        ds.batch(4).assemble(GridMaker(radius_type_indexed=True), [0, 17, 18])


def test_job_table_unstaged_group_counts():
    """More (example, channel) groups than k_job_build stages in shared memory
    (12032): 180 examples x 70 channels.  The device table still equals the
    host builder's entry for entry, and the forward equals the host-packed one."""
    from conftest import random_coordinate_set
    from paper_1912_04822_b200 import Example, GridMaker, _native
    from paper_1912_04822_b200.dataset import DeviceDataset

    rng = np.random.default_rng(11)
    exs = [Example(coord_sets=[random_coordinate_set(rng, int(rng.integers(0, 12)), 14, 6.0)
                               for _ in range(5)]) for _ in range(180)]
    ds = DeviceDataset(exs)
    assert ds.nchannels == 70 and 180 * 70 > 12032
    gm = GridMaker(resolution=1.0, dimension=12.0)
    ids = rng.permutation(180)
    ab = ds.batch(180).assemble(gm, ids)
    pb = gm.pack([exs[i] for i in ids])
    torch.cuda.synchronize()
    N, C = pb.nexamples, pb.nchannels
    p = gm._gm_params(gm.points_per_side())
    co = np.ascontiguousarray(_host_array(pb, "chan_off", N * (C + 1)))
    L = _native.lib()
    cnt = L.gm_forward_jobs(ctypes.byref(p), N, C, co.ctypes.data, None, 0)
    jobs = np.zeros((cnt, 4), np.int32)
    L.gm_forward_jobs(ctypes.byref(p), N, C, co.ctypes.data, jobs.ctypes.data, cnt)
    assert ab._gm.nfwd_jobs == cnt
    np.testing.assert_array_equal(ab._jobs[:cnt].cpu().numpy(), jobs)
    out, _ = gm.forward_packed(ab)
    out2, _ = gm.forward_packed(pb)
    assert torch.equal(out, out2)

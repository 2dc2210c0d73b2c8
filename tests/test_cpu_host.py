"""CPU-only checks: the C ABI library loads and exports every declared
symbol, the host-side mirror (geometry, validation, containers, packing)
behaves like the reference.  No compute call needs a GPU here."""

import math
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def test_library_exports_every_header_symbol():
    from paper_1912_04822_b200 import _native

    header = (ROOT / "include" / "gridmaker_b200.h").read_text()
    header = re.sub(r"/\*.*?\*/", "", header, flags=re.S)
    declared = set(re.findall(r"\b(gm_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    L = _native.load_library()
    for name in sorted(declared):
        assert hasattr(L, name), f"{name} declared in the header but not exported"
    assert set(_native.EXPORTS) == declared


def test_abi_struct_sizes_match_bindings():
    import ctypes

    from paper_1912_04822_b200 import _native

    L = _native.load_library()
    assert L.gm_struct_size(0) == ctypes.sizeof(_native.GmParams)
    assert L.gm_struct_size(1) == ctypes.sizeof(_native.GmBatch)
    assert L.gm_struct_size(2) == ctypes.sizeof(_native.GmDataset)
    assert L.gm_struct_size(3) == ctypes.sizeof(_native.GmCapacity)
    assert L.gm_struct_size(4) == ctypes.sizeof(_native.GmPackSet)
    assert L.gm_struct_size(5) == ctypes.sizeof(_native.GmPackLayout)
    assert L.gm_struct_size(6) == ctypes.sizeof(_native.GmPackInfo)
    assert L.gm_struct_size(7) == ctypes.sizeof(_native.GmPackVSet)
    assert L.gm_struct_size(8) == ctypes.sizeof(_native.GmPackVLayout)
    assert L.gm_version().startswith(b"gridmaker_b200")


def test_workspace_bytes_monotone():
    from paper_1912_04822_b200 import _native

    L = _native.load_library()
    a = L.gm_workspace_bytes(10, 10, 1, 28)
    b = L.gm_workspace_bytes(1000, 5000, 50, 28)
    assert 0 < a < b
    assert b >= 1000 * 24 + 5000 * (64 + 32 + 4 + 64 + 32) + 50 * 29 * 4


def test_invalid_arguments_return_status_not_crash():
    import ctypes

    from paper_1912_04822_b200 import _native

    L = _native.load_library()
    assert L.gm_prepare(None, None, None, 0, None) == 1
    assert b"params" in L.gm_last_error()
    p = _native.GmParams(resolution=0.5, npts=48, radius_multiple=1.5)
    assert L.gm_forward(ctypes.byref(p), None, None, None, None) == 1
    assert b"batch" in L.gm_last_error()


def test_no_cpu_fallback_without_device(monkeypatch):
    import torch

    from paper_1912_04822_b200 import DeviceError, GridMaker
    from paper_1912_04822_b200.synthetic import ligand_only

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(DeviceError):
        GridMaker().forward(ligand_only())


# ---------------------------------------------------------------- geometry

def test_draw_transforms_matches_sequential_make_transform():
    from paper_1912_04822_b200 import geom

    centers = np.random.default_rng(0).uniform(-3, 3, (7, 3))
    for rot, tr in ((True, 2.0), (True, 0.0), (False, 1.5)):
        r1, r2 = np.random.default_rng(11), np.random.default_rng(11)
        seq = [geom.make_transform(c, tr, rot, r1) for c in centers]
        vec = geom.draw_transforms(centers, tr, rot, r2)
        for a, b in zip(seq, vec):
            np.testing.assert_array_equal(a.packed(), b.packed())
        assert r1.random() == r2.random()  # same stream position afterwards


def test_draw_transform_array_bit_identical():
    from paper_1912_04822_b200 import geom

    for seed in range(3):
        centers = np.random.default_rng(seed).uniform(-3, 3, (64, 3))
        for rot, tr in ((True, 2.0), (True, 0.0), (False, 1.5), (False, 0.0)):
            seq = [geom.make_transform(c, tr, rot, r) for r in [np.random.default_rng(seed)]
                   for c in centers]
            arr = geom.draw_transform_array(centers, tr, rot, np.random.default_rng(seed))
            assert len(arr) == 64
            for a, b in zip(seq, arr.packed):
                np.testing.assert_array_equal(a.packed(), b)
            np.testing.assert_array_equal(arr[5].packed(), seq[5].packed())


def test_matmul_order_calibrated():
    from paper_1912_04822_b200 import geom

    assert geom.matmul_order(1) >= 0
    assert geom.matmul_order(50) >= 0


def test_quaternion_basics():
    from paper_1912_04822_b200 import Quaternion, random_unit_quaternion

    q = Quaternion()
    np.testing.assert_allclose(q.rotation_matrix(), np.eye(3), atol=1e-12)
    assert Quaternion(2.0, 0, 0, 0).w == 1.0
    with pytest.raises(ValueError):
        Quaternion(0.0, 0.0, 0.0, 0.0)
    s = math.sqrt(2.0) / 2.0
    np.testing.assert_allclose(Quaternion(s, 0, 0, s).rotate([1.0, 0, 0]), [0, 1, 0], atol=1e-7)
    r = random_unit_quaternion(np.random.default_rng(7))
    np.testing.assert_allclose(r.rotation_matrix() @ r.conjugate().rotation_matrix(), np.eye(3),
                               atol=1e-12)


def test_mean_rotation_angle_uniform_so3():
    from paper_1912_04822_b200 import random_unit_quaternion

    rng = np.random.default_rng(2024)
    angles = [random_unit_quaternion(rng).angle for _ in range(10_000)]
    mean_deg = math.degrees(sum(angles) / len(angles))
    assert abs(mean_deg - math.degrees(math.pi / 2 + 2 / math.pi)) < 2.0


def test_transform_rigid_and_inverse():
    from paper_1912_04822_b200 import make_transform

    rng = np.random.default_rng(5)
    for _ in range(20):
        x = rng.uniform(-10, 10, (9, 3))
        t = make_transform(rng.uniform(-3, 3, 3), 4.0, True, rng)
        y = t.forward(x)
        d0 = np.linalg.norm(x[:, None] - x[None], axis=-1)
        d1 = np.linalg.norm(y[:, None] - y[None], axis=-1)
        assert np.abs(d0 - d1).max() < 1e-4
        np.testing.assert_allclose(t.inverse().forward(y), x, atol=1e-4)


def test_transform_matches_reference_fixture():
    from golden_io import load
    from paper_1912_04822_b200 import Quaternion, Transform

    d = load("transforms")
    for i, pk in enumerate(d["packs"]):
        R = pk[:9].reshape(3, 3)
        t = Transform(Quaternion(), pk[9:12], pk[12:15])
        object.__setattr__(t, "rotation", _FixedRotation(R))
        np.testing.assert_array_equal(t.forward(d[f"x{i}"].astype(np.float64)), d[f"y{i}"])


class _FixedRotation:
    def __init__(self, R):
        self.R = R

    def rotation_matrix(self):
        return self.R


def test_make_transform_validation():
    from paper_1912_04822_b200 import IDENTITY_QUATERNION, make_transform

    t = make_transform((0, 0, 0), 0.0, False, np.random.default_rng(0))
    assert t.rotation == IDENTITY_QUATERNION and not t.translation.any()
    with pytest.raises(ValueError):
        make_transform((0, 0, 0), -1.0, False, np.random.default_rng(0))
    rng = np.random.default_rng(9)
    for _ in range(50):
        assert (np.abs(make_transform((0, 0, 0), 2.0, False, rng).translation) <= 2.0).all()


# ---------------------------------------------------------------- containers

def test_coordinate_set_invariants():
    from paper_1912_04822_b200 import CoordinateSet, make_vector_types

    with pytest.raises(ValueError):
        CoordinateSet(coords=np.zeros((2, 3)), radii=[1.0], num_types=1, type_index=[0, 0])
    with pytest.raises(ValueError):
        CoordinateSet(coords=np.zeros((1, 3)), radii=[0.0], num_types=1, type_index=[0])
    with pytest.raises(ValueError):
        CoordinateSet(coords=np.zeros((1, 3)), radii=[1.0], num_types=1)
    with pytest.raises(ValueError):
        CoordinateSet(coords=np.zeros((1, 3)), radii=[1.0], num_types=2, type_index=[2])
    with pytest.raises(ValueError):
        CoordinateSet(coords=[[np.nan, 0, 0]], radii=[1.0], num_types=1, type_index=[0])
    cs = CoordinateSet(coords=[[1, 2, 3], [3, 2, 1]], radii=[1, 2], num_types=3,
                       type_index=[0, 2])
    np.testing.assert_array_equal(cs.centroid(), [2.0, 2.0, 2.0])
    v = make_vector_types(cs)
    np.testing.assert_array_equal(v.type_vector, [[1, 0, 0], [0, 0, 1]])
    with pytest.raises(ValueError):
        make_vector_types(v)


def test_gridmaker_host_geometry_and_params():
    from paper_1912_04822_b200 import GridMaker

    for res, dim, want in ((0.5, 23.5, 48), (1.0, 23.0, 24), (0.5, 0.0, 1), (0.25, 6.0, 25),
                           (0.25, 23.75, 96)):
        assert GridMaker(resolution=res, dimension=dim).points_per_side() == want
    with pytest.raises(ValueError):
        GridMaker(resolution=0.0).points_per_side()
    gm = GridMaker()
    assert gm.density(0.0, 1.0) == 1.0
    assert abs(gm.density(1.0, 1.0) - math.exp(-2)) < 1e-12
    assert gm.density(1.5, 1.0) == 0.0 and gm.density(1.499, 1.0) > 0.0
    assert GridMaker(binary=True).density(0.99, 1.0) == 1.0
    np.testing.assert_array_equal(gm.grid_origin((0, 0, 0)), [-11.75] * 3)
    params = GridMaker(resolution=1.0, binary=True).get_params()
    assert GridMaker().set_params(**params).get_params() == params
    with pytest.raises(ValueError):
        GridMaker().set_params(voxels=3)
    with pytest.raises(ValueError):
        GridMaker(radius_scale=-1.0).fit()
    # estimator-style: pickles / deep-copies as its parameters, without the
    # numpy API's per-thread pack cache (device buffers, unpicklable handles)
    import copy
    import pickle
    import threading

    gm = GridMaker(resolution=0.25, dimension=10.0)
    gm.__dict__["_pack_cache"] = {threading.get_ident(): (None, threading.Lock())}
    for clone in (pickle.loads(pickle.dumps(gm)), copy.deepcopy(gm)):
        assert clone.get_params() == gm.get_params() and "_pack_cache" not in clone.__dict__


@pytest.mark.parametrize("grm", [0.5, 1.0, 1.5, 2.0])
@pytest.mark.parametrize("r", [0.5, 1.0, 1.9, 2.2])
def test_density_c1_continuity(grm, r):
    from paper_1912_04822_b200 import GridMaker

    gm = GridMaker(gaussian_radius_multiple=grm)
    d0, eps = grm * r, 1e-9
    assert abs(gm.density(d0 - eps, r) - gm.density(d0 + eps, r)) < 1e-6
    assert abs(gm.density_slope(d0 - eps, r) - gm.density_slope(d0 + eps, r)) < 1e-5


def test_batch_validation_before_device():
    """The reference's argument errors are raised before any device work."""
    from conftest import random_coordinate_set
    from paper_1912_04822_b200 import Example, GridMaker, make_vector_types

    rng = np.random.default_rng(0)
    gm = GridMaker()
    with pytest.raises(ValueError):
        gm.forward_batch([])
    with pytest.raises(TypeError):
        gm.forward_batch([object()])
    a = Example([random_coordinate_set(rng, 3, 2)])
    b = Example([random_coordinate_set(rng, 3, 3)])
    with pytest.raises(ValueError):
        gm.forward_batch([a, b])
    v = Example([make_vector_types(random_coordinate_set(rng, 3, 2))])
    with pytest.raises(ValueError):
        gm.forward_batch([a, v])
    with pytest.raises(ValueError):
        gm.forward_batch([a], out=np.zeros((1, 3, 48, 48, 48), np.float32))
    with pytest.raises(TypeError):
        gm.forward_batch([a], out=np.zeros((1, 2, 48, 48, 48), np.float64))
    with pytest.raises(ValueError):
        gm.forward_batch([a], centers=np.zeros((2, 3)))
    with pytest.raises(TypeError):
        gm.forward(a)


def test_all_empty_batch_consumes_no_random_numbers():
    """voxelizer.py:351-352: a batch of empty sets returns before any
    make_transform call, so the caller's generator is untouched."""
    from paper_1912_04822_b200 import CoordinateSet, Example, GridMaker

    empty = CoordinateSet(coords=np.zeros((0, 3), np.float32), radii=np.zeros(0, np.float32),
                          num_types=3, type_index=np.zeros(0, np.int64))
    gm = GridMaker(dimension=4.0)
    rng = np.random.default_rng(42)
    before = rng.bit_generator.state
    grid, xf = gm.forward_batch([Example([empty]), Example([empty])], random_rotation=True,
                                random_translation=2.0, rng=rng, return_transforms=True)
    assert rng.bit_generator.state == before
    assert xf is None
    assert grid.shape == (2, 3, 9, 9, 9) and not grid.any()


def test_packing_layout_cpu():
    import torch

    from paper_1912_04822_b200 import synthetic
    from paper_1912_04822_b200.packing import PackedBatch

    exs = synthetic.batch(3, seed=2, vector=True)
    sets = [ex.coord_sets for ex in exs]
    pb = PackedBatch(sets, 28, True, 1.1, True, torch.device("cpu"))
    assert pb.natoms == 3 * 1030 and pb.nsets == 6
    host = pb.host.numpy()

    def arr(name):
        off, dt, shape = pb.offsets[name]
        n = int(np.prod(shape))
        return host[off:off + n * dt.itemsize].view(dt).reshape(shape)

    ia, ic, iw = arr("item_atom"), arr("item_channel"), arr("item_weight")
    assert pb.nitems == ia.shape[0] == sum(int((cs.type_vector != 0).sum()) for s in sets for cs in s)
    assert (np.diff(ia) >= 0).all()  # atom-major order
    es, ee = arr("ex_item_start"), arr("ex_item_end")
    assert es[0] == 0 and ee[-1] == pb.nitems and (es[1:] == ee[:-1]).all()
    # radius_type_indexed: item radius = type radius * scale
    tr = arr("item_radius")
    np.testing.assert_allclose(tr, synthetic.TYPE_RADII[ic].astype(np.float64) * 1.1)
    np.testing.assert_array_equal(arr("set_choff"), [0, 14] * 3)
    np.testing.assert_array_equal(pb.default_centers[0], exs[0].coord_sets[1].centroid())


def test_vector_item_windex_maps_items_to_weight_rows():
    """PackedBatch.item_windex (autograd weight refresh) points every forward
    item at its entry of the packed weight rows."""
    from paper_1912_04822_b200 import synthetic
    from paper_1912_04822_b200.packing import PackedBatch

    exs = synthetic.batch(3, seed=4, vector=True)
    pb = PackedBatch([ex.coord_sets for ex in exs], 28, True, 1.0, False, "cpu")
    host = {}
    for name in ("weights", "item_weight"):
        off, dt, shape = pb.offsets[name]
        n = int(np.prod(shape))
        host[name] = pb.host.numpy()[off:off + n * np.dtype(dt).itemsize].view(dt)
    assert pb.item_windex.shape == (pb.nitems,)
    np.testing.assert_array_equal(host["weights"][pb.item_windex], host["item_weight"])
    assert pb.atom_example.shape == (pb.natoms,)


def test_forward_job_table_covers_every_tile_once():
    """gm_forward_jobs (host side of the C ABI): every tile of a channel with
    items exactly once, one job per GM_FWD_ZGROUP group of a zero slab, the
    (plane, row) field consistent with the tile index."""
    import ctypes

    from paper_1912_04822_b200 import GridMaker, _native, synthetic
    from paper_1912_04822_b200.packing import PackedBatch

    exs = synthetic.batch(3, seed=2)
    pb = PackedBatch([ex.coord_sets for ex in exs], 28, False, 1.0, False, "cpu")
    lib = _native.load_library()
    for res, dim in ((0.5, 23.5), (0.25, 23.75)):
        gm = GridMaker(resolution=res, dimension=dim)
        D = gm.points_per_side()
        p = gm._gm_params(D)
        off = pb.offsets["chan_off"][0]
        n = pb.nexamples * (pb.nchannels + 1)
        co = np.ascontiguousarray(pb.host.numpy()[off:off + 4 * n].view(np.int32))
        cnt = lib.gm_forward_jobs(ctypes.byref(p), 3, 28, co.ctypes.data, None, 0)
        jobs = np.zeros((cnt, 4), np.int32)
        assert lib.gm_forward_jobs(ctypes.byref(p), 3, 28, co.ctypes.data, jobs.ctypes.data,
                                   cnt) == cnt
        co2 = co.reshape(3, 29)
        # gm_batch.max_seg_items / segs: the largest group and the groups with items
        assert pb.max_seg_items == int(np.diff(co2, axis=1).max())
        assert pb.nsegs == int((np.diff(co2, axis=1) > 0).sum())
        nonzero = {(e, c) for e in range(3) for c in range(28) if co2[e, c + 1] > co2[e, c]}
        seen = {}
        ntj = None
        for ec, cs, ce, ij in jobs:
            e, c = ec & 0xffff, ec >> 16
            i0, j0 = ij & 0xffff, ij >> 16
            assert 0 <= i0 < D and 0 <= j0 < D
            assert (cs, ce) == (co2[e, c], co2[e, c + 1])  # the static item range
            seen.setdefault((e, c), []).append((i0, j0))
        # tiles as (plane, row band) pairs -> dense tile indices
        rows = sorted({j for v in seen.values() for (_, j) in v})
        planes = sorted({i for v in seen.values() for (i, _) in v})
        ntj = len(rows)
        seen = {k: [planes.index(i) * ntj + rows.index(j) for (i, j) in v] for k, v in seen.items()}
        ntiles = max(max(v) for v in seen.values()) + 1
        for (e, c), ts in seen.items():
            if (e, c) in nonzero:
                assert sorted(ts) == list(range(ntiles))
            else:
                # one job per group of GM_FWD_ZGROUP tiles: 0, g, 2g, ... < ntiles
                ts = sorted(ts)
                g = ts[1] - ts[0] if len(ts) > 1 else ntiles
                assert ts == list(range(0, ntiles, g)) and g >= 8
        assert len(seen) == 3 * 28


def test_thread_control_api():
    """set_num_threads / get_num_threads (voxelizer.py:33-52): validation and
    the returned count."""
    import pytest

    from paper_1912_04822_b200 import get_num_threads, set_num_threads

    n0 = get_num_threads()
    assert n0 >= 1
    assert set_num_threads(1) == 1 == get_num_threads()
    with pytest.raises(ValueError):
        set_num_threads(0)
    set_num_threads(n0)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_native_packer_equals_numpy_packing(seed, monkeypatch):
    """gm_pack_index_host (csrc/pack.cu) writes the numpy packing's arrays:
    every array byte for byte, except the backward launch order, which must
    be a permutation grouping each (example, channel) slab's atoms together.
    Odd shapes included: empty and single-atom sets, an example without atoms."""
    import torch

    import paper_1912_04822_b200.packing as packing
    from conftest import random_coordinate_set
    from paper_1912_04822_b200 import synthetic

    rng = np.random.default_rng(seed)
    exs = [ex.coord_sets for ex in synthetic.batch(4, seed=seed)]
    for k in range(4):
        exs.append([random_coordinate_set(rng, [0, 1, 7, 0][k], 14, 9.0),
                    random_coordinate_set(rng, [5, 0, 1, 0][k], 14, 4.0)])
    scale = [1.0, 0.7, 1.3][seed]

    def build(native):
        monkeypatch.setattr(packing, "_NATIVE_PACK", native)
        return packing.PackedBatch(exs, 28, False, scale, False, torch.device("cpu"))

    a, b = build(True), build(False)
    for attr in ("natoms", "nsets", "nitems", "nsegs", "max_seg_items", "max_example_items"):
        assert getattr(a, attr) == getattr(b, attr), attr
    np.testing.assert_array_equal(a.default_centers, b.default_centers)
    np.testing.assert_array_equal(a.atom_example, b.atom_example)
    assert [(e, c, id(cs), a0) for e, c, cs, a0, _ in a.placed] == \
        [(e, c, id(cs), a0) for e, c, cs, a0, _ in b.placed]

    def arr(pb, name):
        off, dt, shape = pb.offsets[name]
        n = int(np.prod(shape))
        return pb.host.numpy()[off:off + n * dt.itemsize].view(dt).reshape(shape)

    for name in ("coords32", "atom_radius", "atom_set", "atom_type", "set_start", "set_end",
                 "set_example", "set_choff", "set_t", "ex_item_start", "ex_item_end",
                 "item_perm", "chan_off", "segs"):
        np.testing.assert_array_equal(arr(a, name), arr(b, name), err_msg=name)
    ra = arr(a, "slot_rec").view(packing._SLOT_DTYPE)
    rb = arr(b, "slot_rec").view(packing._SLOT_DTYPE)
    for f in ("x", "y", "z", "atom", "ch", "ex", "single", "r"):
        np.testing.assert_array_equal(ra[f], rb[f], err_msg=f)
    bs = arr(a, "bwd_slot")
    assert np.array_equal(np.sort(bs), np.arange(a.natoms))
    np.testing.assert_array_equal(ra["bslot"], bs[ra["atom"]])
    # slab grouping: in launch order, each (example, channel) slab is contiguous
    slab = a.atom_example.astype(np.int64) * 28 + arr(a, "set_choff")[arr(a, "atom_set")] + \
        arr(a, "atom_type")
    launch = slab[np.argsort(bs)]
    assert (np.diff(launch) >= 0).all()


def test_native_packer_without_atoms():
    """A batch whose sets are all empty packs (no slot records, no launch order)."""
    import torch

    from conftest import random_coordinate_set
    from paper_1912_04822_b200.packing import PackedBatch

    rng = np.random.default_rng(0)
    exs = [[random_coordinate_set(rng, 0, 3, 4.0), random_coordinate_set(rng, 0, 2, 4.0)]] * 2
    pb = PackedBatch(exs, 5, False, 1.0, False, torch.device("cpu"))
    assert pb.natoms == 0 and pb.nsegs == 0 and "slot_rec" not in pb.offsets


@pytest.mark.parametrize("rti", [False, True])
def test_native_vector_packer_equals_numpy_packing(rti, monkeypatch):
    """gm_pack_vector_host writes the numpy vector packing's arrays (weights,
    type radii, nonzero-weight items, static grouping), the same item_windex
    and placements; its launch order keeps each example's atoms together."""
    import torch

    import paper_1912_04822_b200.packing as packing
    from conftest import random_coordinate_set
    from paper_1912_04822_b200 import make_vector_types, synthetic

    from paper_1912_04822_b200.coordsets import CoordinateSet

    rng = np.random.default_rng(4)
    exs = [ex.coord_sets for ex in synthetic.batch(4, seed=4, vector=True)]
    tr = synthetic.TYPE_RADII.astype(np.float32)

    def odd(n):  # vector-typed set with type radii (empty / single-atom ones included)
        v = make_vector_types(random_coordinate_set(rng, n, 14, 8.0))
        return CoordinateSet(coords=v.coords, radii=v.radii, num_types=14,
                             type_vector=v.type_vector, type_radii=tr)

    for k in range(3):
        exs.append([odd([0, 1, 9][k]), odd([6, 0, 1][k])])

    def build(native):
        monkeypatch.setattr(packing, "_NATIVE_PACK", native)
        return packing.PackedBatch(exs, 28, True, 1.2, rti, torch.device("cpu"))

    a, b = build(True), build(False)
    for attr in ("natoms", "nsets", "nitems", "nweights", "nsegs", "max_seg_items",
                 "max_example_items"):
        assert getattr(a, attr) == getattr(b, attr), attr
    np.testing.assert_array_equal(a.item_windex, b.item_windex)
    np.testing.assert_array_equal(a.atom_example, b.atom_example)
    assert [(e, c, a0, w) for e, c, _, a0, w in a.placed] == \
        [(e, c, a0, w) for e, c, _, a0, w in b.placed]

    def arr(pb, name):
        off, dt, shape = pb.offsets[name]
        n = int(np.prod(shape))
        return pb.host.numpy()[off:off + n * dt.itemsize].view(dt).reshape(shape)

    for name in ("coords32", "atom_radius", "atom_set", "set_start", "set_end", "set_example",
                 "set_choff", "set_t", "set_wstart", "set_trstart", "weights", "type_radius",
                 "item_atom", "item_channel", "item_weight", "item_radius", "ex_item_start",
                 "ex_item_end", "item_perm", "chan_off", "segs"):
        np.testing.assert_array_equal(arr(a, name), arr(b, name), err_msg=name)
    bs = arr(a, "bwd_slot")
    assert np.array_equal(np.sort(bs), np.arange(a.natoms))
    assert (np.diff(a.atom_example[np.argsort(bs)]) >= 0).all()

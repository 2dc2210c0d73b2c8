"""GPU parity: the CUDA path (through GridMaker -> C ABI) against the golden
fixtures of the live reference and the CPU oracle, on the same inputs."""

import numpy as np
import pytest

import oracle
from golden_io import (BATCH_FIXTURES, SINGLE_FIXTURES, VECTOR_FIXTURES, aug_from,
                       dense_from_sparse, examples_from, expected_grid, load, params_from,
                       sets_from, unpack_bits)
from parity import assert_close, to_numpy

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def gm_of(params, **kw):
    from paper_1912_04822_b200 import GridMaker

    return GridMaker(**params, **kw)


@pytest.mark.parametrize("name", SINGLE_FIXTURES)
def test_single_forward_golden(name):
    d = load(name)
    grid = gm_of(params_from(d)).forward(sets_from(d)[0], center=d["center"])
    assert_close(grid, d["grid"], what=name)
    if name.startswith("fwd_index"):
        # the reference's own absolute gate (test_voxelizer.py:146)
        assert np.abs(grid.astype(np.float64) - d["grid"]).max() < 1e-6


@pytest.mark.parametrize("name", BATCH_FIXTURES + VECTOR_FIXTURES)
def test_batch_forward_golden(name):
    d = load(name)
    p = params_from(d)
    grid = gm_of(p).forward_batch(examples_from(d), **aug_from(d))
    want = expected_grid(d)
    if p["binary"]:
        np.testing.assert_array_equal(grid, want)
    else:
        assert_close(grid, want, what=name)


def test_backward_index_golden():
    d = load("bwd_index")
    cg, tg = gm_of(params_from(d)).backward(sets_from(d)[0], d["grid_grad"], center=d["center"])
    assert tg is None
    assert_close(cg, d["coord_grad"], what="bwd_index")


@pytest.mark.parametrize("rti", [0, 1])
def test_backward_vector_golden(rti):
    d = load(f"bwd_vector_rti{rti}")
    cg, tg = gm_of(params_from(d)).backward(sets_from(d)[0], d["grid_grad"], center=d["center"])
    assert_close(cg, d["coord_grad"], what="coord")
    assert_close(tg, d["type_grad"], what="type")


def test_c2_example_golden_offset_frame():
    d = load("c2_example")
    exs = examples_from(d)
    gm = gm_of({})
    grid = gm.forward_batch(exs)
    want = dense_from_sparse(d)
    assert_close(grid, want, what="c2 forward")
    res = gm.backward_batch(exs, want)
    assert_close(res[0][0][0], d["coord_grad_rec"], what="c2 receptor grad")
    assert_close(res[0][1][0], d["coord_grad_lig"], what="c2 ligand grad")


def test_c3_example_golden_bit_exact():
    d = load("c3_example")
    grid = gm_of({"binary": True}).forward_batch(
        examples_from(d), random_rotation=True, random_translation=2.0,
        rng=np.random.default_rng(int(d["aug_seed"])))
    np.testing.assert_array_equal(grid, unpack_bits(d))


# ------------------------------------------------------------ full-size vs oracle

def _synthetic(n, seed, vector=False, offset=None):
    from paper_1912_04822_b200 import synthetic

    return synthetic.batch(n, seed=seed, vector=vector, offset=offset)


@pytest.mark.parametrize("offset", [False, True])
def test_c2_batch_fwd_bwd_vs_oracle(offset):
    from paper_1912_04822_b200 import synthetic

    exs = _synthetic(50, 2, offset=synthetic.PDB_OFFSET if offset else None)
    gm = gm_of({})
    go = oracle.GridOracle()
    grid, xf = gm.forward_batch(exs, random_rotation=True, random_translation=2.0,
                                rng=np.random.default_rng(3), return_transforms=True)
    ref = go.forward_batch(exs, random_rotation=True, random_translation=2.0,
                           rng=np.random.default_rng(3))
    assert_close(grid, ref, what="C2 forward")
    gg = np.random.default_rng(7).standard_normal(grid.shape, dtype=np.float32)
    got = gm.backward_batch(exs, gg, transforms=xf)
    cgs, _ = go.backward_batch(exs, gg, random_rotation=True, random_translation=2.0,
                               rng=np.random.default_rng(3))
    flat_got = np.concatenate([c for ex in got for (c, t) in ex])
    assert_close(flat_got, np.concatenate(cgs), what="C2 backward (N(0,1) grad)")
    # physically shaped gradient: d(1/2 |grid|^2)/d grid = grid
    got2 = gm.backward_batch(exs, ref, transforms=xf)
    cgs2, _ = go.backward_batch(exs, ref, random_rotation=True, random_translation=2.0,
                                rng=np.random.default_rng(3))
    assert_close(np.concatenate([c for ex in got2 for (c, t) in ex]), np.concatenate(cgs2),
                 what="C2 backward (grid grad)")


def test_c3_batch_binary_bit_exact_vs_oracle():
    exs = _synthetic(50, 2)
    gm = gm_of({"binary": True})
    go = oracle.GridOracle(binary=True)
    grid = gm.forward_batch(exs, random_rotation=True, random_translation=2.0,
                            rng=np.random.default_rng(0))
    ref = go.forward_batch(exs, random_rotation=True, random_translation=2.0,
                           rng=np.random.default_rng(0))
    np.testing.assert_array_equal(grid, ref)


@pytest.mark.parametrize("rti", [False, True])
def test_c4_vector_fwd_bwd_vs_oracle(rti):
    exs = _synthetic(12, 4, vector=True)
    gm = gm_of({"radius_type_indexed": rti})
    go = oracle.GridOracle(radius_type_indexed=rti)
    grid, xf = gm.forward_batch(exs, random_rotation=True, rng=np.random.default_rng(5),
                                return_transforms=True)
    ref = go.forward_batch(exs, random_rotation=True, rng=np.random.default_rng(5))
    assert_close(grid, ref, what="C4 forward")
    gg = np.random.default_rng(7).standard_normal(grid.shape, dtype=np.float32)
    got = gm.backward_batch(exs, gg, transforms=xf)
    cgs, tgs = go.backward_batch(exs, gg, random_rotation=True, rng=np.random.default_rng(5))
    assert_close(np.concatenate([c for ex in got for (c, t) in ex]), np.concatenate(cgs),
                 what="C4 coord grad")
    assert_close(np.concatenate([t.reshape(-1) for ex in got for (c, t) in ex]),
                 np.concatenate([t.reshape(-1) for t in tgs]), what="C4 type grad")


def test_c4_vector_binary_vs_oracle():
    exs = _synthetic(6, 4, vector=True)
    gm = gm_of({"binary": True})
    go = oracle.GridOracle(binary=True)
    grid = gm.forward_batch(exs, random_rotation=True, rng=np.random.default_rng(6))
    ref = go.forward_batch(exs, random_rotation=True, rng=np.random.default_rng(6))
    np.testing.assert_array_equal(grid, ref)


def test_c5_fine_grid_vs_oracle():
    exs = _synthetic(4, 2)
    gm = gm_of({"resolution": 0.25, "dimension": 23.75})
    assert gm.points_per_side() == 96
    go = oracle.GridOracle(resolution=0.25, dimension=23.75)
    grid, xf = gm.forward_batch(exs, random_rotation=True, rng=np.random.default_rng(8),
                                return_transforms=True)
    ref = go.forward_batch(exs, random_rotation=True, rng=np.random.default_rng(8))
    assert_close(grid, ref, what="C5 forward")
    gg = np.random.default_rng(9).standard_normal(grid.shape, dtype=np.float32)
    got = gm.backward_batch(exs, gg, transforms=xf)
    cgs, _ = go.backward_batch(exs, gg, random_rotation=True, rng=np.random.default_rng(8))
    assert_close(np.concatenate([c for ex in got for (c, t) in ex]), np.concatenate(cgs),
                 what="C5 backward")


@pytest.mark.parametrize("dim,res", [(8.0, 0.5), (6.0, 0.25), (11.3, 0.7), (0.0, 0.5)])
def test_odd_grid_sizes_vs_oracle(dim, res, rng):
    from conftest import random_coordinate_set
    from paper_1912_04822_b200 import Example

    exs = [Example(coord_sets=[random_coordinate_set(rng, 20, 3, 5.0),
                               random_coordinate_set(rng, 3, 2, 2.0)]) for _ in range(3)]
    for binary in (False, True):
        gm = gm_of({"resolution": res, "dimension": dim, "binary": binary})
        go = oracle.GridOracle(resolution=res, dimension=dim, binary=binary)
        grid = gm.forward_batch(exs, random_rotation=True, rng=np.random.default_rng(1))
        ref = go.forward_batch(exs, random_rotation=True, rng=np.random.default_rng(1))
        if binary:
            np.testing.assert_array_equal(grid, ref)
        else:
            assert_close(grid, ref, what=f"D={gm.points_per_side()}")


def test_single_atom_sets_binary_rotation_bit_exact(rng):
    """Sets of one atom take numpy's N=1 matmul path (gemv order)."""
    from conftest import random_coordinate_set
    from paper_1912_04822_b200 import Example

    exs = [Example(coord_sets=[random_coordinate_set(rng, 1, 2, 4.0),
                               random_coordinate_set(rng, 2, 2, 4.0)]) for _ in range(40)]
    gm = gm_of({"binary": True, "dimension": 12.0})
    go = oracle.GridOracle(binary=True, dimension=12.0)
    grid = gm.forward_batch(exs, random_rotation=True, random_translation=1.0,
                            rng=np.random.default_rng(2))
    ref = go.forward_batch(exs, random_rotation=True, random_translation=1.0,
                           rng=np.random.default_rng(2))
    np.testing.assert_array_equal(grid, ref)


def test_device_tensor_out_and_determinism():
    exs = _synthetic(8, 2)
    from paper_1912_04822_b200 import GridMaker

    gm = GridMaker()
    out = torch.empty((8, 28, 48, 48, 48), device="cuda")
    got = gm.forward_batch(exs, out=out)
    assert got is out
    again = gm.forward_batch(exs)
    np.testing.assert_array_equal(to_numpy(out), again)
    # a slab does not depend on its neighbours in the batch
    solo = gm.forward_batch(exs[3:4])
    np.testing.assert_array_equal(solo[0], again[3])


@pytest.mark.parametrize("binary", [False, True])
def test_boxes_wider_than_32_voxels(binary, rng):
    """res 0.1 A: an atom's box spans ~60 voxels per axis, exercising the
    forward's >32-column path and the backward's sub-box walk."""
    from conftest import random_coordinate_set
    from paper_1912_04822_b200 import Example

    exs = [Example(coord_sets=[random_coordinate_set(rng, 3, 2, 1.5)]) for _ in range(2)]
    gm = gm_of({"resolution": 0.1, "dimension": 7.9, "binary": binary})  # D = 80
    go = oracle.GridOracle(resolution=0.1, dimension=7.9, binary=binary)
    grid, xf = gm.forward_batch(exs, random_rotation=True, rng=np.random.default_rng(4),
                                return_transforms=True)
    ref = go.forward_batch(exs, random_rotation=True, rng=np.random.default_rng(4))
    if binary:
        np.testing.assert_array_equal(grid, ref)
        return
    assert_close(grid, ref, what="wide-box forward")
    gg = np.random.default_rng(5).standard_normal(grid.shape, dtype=np.float32)
    got = gm.backward_batch(exs, gg, transforms=xf)
    cgs, _ = go.backward_batch(exs, gg, random_rotation=True, rng=np.random.default_rng(4))
    assert_close(np.concatenate([c for ex in got for (c, t) in ex]), np.concatenate(cgs),
                 what="wide-box backward")


def test_vector_many_channels_per_set(rng):
    """> 16 channels in a set takes the per-channel vector backward path."""
    from paper_1912_04822_b200 import CoordinateSet, Example

    n, T = 12, 20
    cs = CoordinateSet(coords=rng.uniform(-3, 3, (n, 3)).astype(np.float32),
                       radii=rng.uniform(1.2, 2.0, n).astype(np.float32), num_types=T,
                       type_vector=(rng.random((n, T)) * (rng.random((n, T)) < 0.3))
                       .astype(np.float32))
    exs = [Example(coord_sets=[cs])]
    gm = gm_of({"dimension": 12.0})
    go = oracle.GridOracle(dimension=12.0)
    grid = gm.forward_batch(exs)
    assert_close(grid, go.forward_batch(exs), what="forward")
    gg = np.random.default_rng(2).standard_normal(grid.shape, dtype=np.float32)
    (cg, tg), = gm.backward_batch(exs, gg)[0]
    wc, wt = go.backward_batch(exs, gg)
    assert_close(cg, wc[0], what="coord")
    assert_close(tg, wt[0], what="type")


@pytest.mark.parametrize("binary", [False, True])
def test_example_too_big_for_smem_staging(binary, rng):
    """6000 (atom, channel) items in one example: the prepare kernel stages
    the records in the workspace instead of shared memory."""
    from paper_1912_04822_b200 import CoordinateSet, Example

    n, T = 600, 10
    cs = CoordinateSet(coords=rng.uniform(-8, 8, (n, 3)).astype(np.float32),
                       radii=rng.uniform(1.2, 2.0, n).astype(np.float32), num_types=T,
                       type_vector=rng.uniform(0.1, 1.0, (n, T)).astype(np.float32))
    exs = [Example(coord_sets=[cs]), Example(coord_sets=[cs])]
    gm = gm_of({"dimension": 16.0, "binary": binary})
    go = oracle.GridOracle(dimension=16.0, binary=binary)
    grid = gm.forward_batch(exs, random_rotation=True, rng=np.random.default_rng(1))
    ref = go.forward_batch(exs, random_rotation=True, rng=np.random.default_rng(1))
    if binary:
        np.testing.assert_array_equal(grid, ref)
    else:
        assert_close(grid, ref, what="global-staged forward")


def test_launch_orders_do_not_change_results(monkeypatch):
    """The forward job table (tile order, skipped zero CTAs) and the backward's
    cost-ordered launch are scheduling only: results are bitwise identical to
    the dense launch in atom order."""
    from paper_1912_04822_b200 import GridMaker, packing, synthetic

    exs = synthetic.batch(6, seed=31)
    gm = GridMaker()
    g1, xf = gm.forward_batch(exs, random_rotation=True, random_translation=2.0,
                              rng=np.random.default_rng(4), return_transforms=True)
    b1 = gm.backward_batch(exs, g1, transforms=xf)
    monkeypatch.setattr(packing, "_NO_JOBS", True)
    monkeypatch.setattr(packing, "_BWD_ORDER", "none")
    g2 = gm.forward_batch(exs, random_rotation=True, random_translation=2.0,
                          rng=np.random.default_rng(4))
    b2 = gm.backward_batch(exs, g1, transforms=xf)
    np.testing.assert_array_equal(g1, g2)
    for e1, e2 in zip(b1, b2):
        for (c1, _), (c2, _) in zip(e1, e2):
            np.testing.assert_array_equal(c1, c2)


def test_job_table_with_dynamic_grouping_path():
    """More examples than the inline prepare takes (GM_INLINE_MAX_EXAMPLES):
    the per-example grouping pass runs and the forward re-reads its ranges."""
    from paper_1912_04822_b200 import GridMaker, synthetic

    rng = np.random.default_rng(32)
    exs = [synthetic.complex_example(rng, n_receptor=40, n_ligand=6) for _ in range(205)]
    gm = gm_of({"dimension": 11.5})
    grid = gm.forward_batch(exs, random_rotation=True, random_translation=2.0,
                            rng=np.random.default_rng(6))
    go = oracle.GridOracle(dimension=11.5)
    ref = go.forward_batch(exs, random_rotation=True, random_translation=2.0,
                           rng=np.random.default_rng(6))
    assert_close(grid, ref, what="205-example batch")


@pytest.mark.parametrize("vector,res,dim", [(False, 0.5, 23.5), (True, 0.5, 23.5),
                                            (False, 0.25, 23.75)])
def test_channels_whose_items_all_miss_the_grid(vector, res, dim):
    """A set whose atoms all lie outside the grid: its channels have items in
    the static grouping but none reaches a voxel (empty boxes), under the job
    table, the plane sort and the backward launch order."""
    from paper_1912_04822_b200 import Example, GridMaker, synthetic

    rng = np.random.default_rng(41)
    exs = []
    for _ in range(3):
        far = synthetic.receptor(rng, 60, 3.0, offset=np.array([80.0, -75.0, 90.0]))
        lig = synthetic.ligand(rng, 12, 3.0)
        if vector:
            far, lig = synthetic.vectorize(far, rng), synthetic.vectorize(lig, rng)
        exs.append(Example(coord_sets=[far, lig], labels=[0.0]))
    gm = GridMaker(resolution=res, dimension=dim)
    grid, xf = gm.forward_batch(exs, random_rotation=True, random_translation=1.0,
                                rng=np.random.default_rng(2), return_transforms=True)
    go = oracle.GridOracle(resolution=res, dimension=dim)
    ref = go.forward_batch(exs, random_rotation=True, random_translation=1.0,
                           rng=np.random.default_rng(2))
    assert not grid[:, :14].any()
    assert_close(grid, ref, what="far-set batch")
    got = gm.backward_batch(exs, ref, transforms=xf)
    cgs, tgs = go.backward_batch(exs, ref, random_rotation=True, random_translation=1.0,
                                 rng=np.random.default_rng(2))
    assert_close(np.concatenate([c for ex in got for (c, _) in ex]), np.concatenate(cgs),
                 what="far-set backward")


@pytest.mark.parametrize("vector", [False, True])
def test_binary_boundary_voxels_bit_exact(vector):
    """Binary occupancy where many voxels sit exactly on (or an ulp from) the
    sphere: atoms on voxel centers with r^2 = k res^2 (k = 1..6), and PDB-like
    offsets -- the f32 fast test must defer every such voxel to the exact f64
    expression."""
    from paper_1912_04822_b200 import CoordinateSet, Example, GridMaker

    res = 0.5
    rng = np.random.default_rng(51)
    sets = []
    for k in range(1, 7):
        n = 20
        ijk = rng.integers(4, 20, size=(n, 3)).astype(np.float64)
        coords = (-5.75 + res * ijk + np.array([41.37, -27.91, 63.05])).astype(np.float32)
        radii = np.full(n, np.sqrt(k) * res, np.float32)
        if vector:
            tv = (rng.random((n, 3)) < 0.6).astype(np.float32) * rng.random((n, 3)).astype(np.float32)
            sets.append(CoordinateSet(coords=coords, radii=radii, num_types=3, type_vector=tv))
        else:
            sets.append(CoordinateSet(coords=coords, radii=radii, num_types=3,
                                      type_index=rng.integers(0, 3, n)))
    exs = [Example(coord_sets=[s], labels=[0.0]) for s in sets]
    center = np.array([41.37, -27.91, 63.05])
    gm = GridMaker(resolution=res, dimension=11.5, binary=True)
    grid = gm.forward_batch(exs, centers=np.tile(center, (len(exs), 1)))
    go = oracle.GridOracle(resolution=res, dimension=11.5, binary=True)
    ref = go.forward_batch(exs, centers=np.tile(center, (len(exs), 1)))
    np.testing.assert_array_equal(grid, ref)


def test_plane_sort_fallback_for_crowded_channels():
    """More items in one channel than the plane sort stages (1024): that
    channel keeps item order and scans its whole range; results match."""
    from paper_1912_04822_b200 import CoordinateSet, Example, GridMaker

    rng = np.random.default_rng(61)
    n = 1500
    coords = rng.uniform(-6, 6, size=(n, 3)).astype(np.float32)
    cs = CoordinateSet(coords=coords, radii=np.full(n, 1.2, np.float32), num_types=3,
                       type_index=np.where(np.arange(n) < 1300, 0, rng.integers(1, 3, n)))
    exs = [Example(coord_sets=[cs], labels=[0.0])]
    gm = GridMaker(resolution=0.125, dimension=11.875)  # D = 96: plane sort enabled
    grid = gm.forward_batch(exs, random_rotation=True, rng=np.random.default_rng(3))
    go = oracle.GridOracle(resolution=0.125, dimension=11.875)
    ref = go.forward_batch(exs, random_rotation=True, rng=np.random.default_rng(3))
    assert_close(grid, ref, what="crowded channel, fine grid")

"""The reference's own hot-path tests, run against the CUDA GridMaker.

Mirrors /root/reference/pkg/tests/test_voxelizer.py (forward single 86-134,
oracle equivalence 137-191, properties 194-235, batch 244-312, backward
315-387, estimator 390-427) and the gridding criteria of
test_acceptance.py (oracle equivalence 75-89, gradient check 122-188,
default shape 191-207, determinism 351-389, transform suite 392-411).
The checker is the independent all-pairs oracle (oracle/allpairs.py).
"""

import numpy as np
import pytest

from conftest import random_coordinate_set
from oracle.allpairs import (central_differences, grid_all_pairs, mask_seams,
                             relative_errors)
from parity import to_numpy

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _gm(**kw):
    from paper_1912_04822_b200 import GridMaker

    return GridMaker(**kw)


def single_atom(position, radius=1.0, num_types=1, index=0):
    from paper_1912_04822_b200 import CoordinateSet

    return CoordinateSet(coords=np.array([position], dtype=np.float32),
                         radii=np.array([radius], dtype=np.float32), num_types=num_types,
                         type_index=np.array([index], dtype=np.int64))


def _two_set_example(rng, n1=6, n2=4, num_types=3):
    from paper_1912_04822_b200 import Example

    return Example(coord_sets=[random_coordinate_set(rng, n1, num_types=num_types, extent=4.0),
                               random_coordinate_set(rng, n2, num_types=num_types, extent=4.0)],
                   labels=[1.0])


# ---------------------------------------------------------------- forward single

def test_atom_on_voxel_center_is_exactly_one():
    grid = _gm().forward(single_atom((-0.25, -0.25, -0.25), 1.0, 3, 1), center=(0.0, 0.0, 0.0))
    assert grid.shape == (3, 48, 48, 48)
    assert grid[1, 23, 23, 23] == 1.0
    assert not grid[0].any() and not grid[2].any()


def test_empty_atom_set_and_far_atom():
    from paper_1912_04822_b200 import CoordinateSet

    empty = CoordinateSet(coords=np.zeros((0, 3)), radii=np.zeros(0), num_types=4,
                          type_index=np.zeros(0, dtype=np.int64))
    g = _gm().forward(empty, center=(0, 0, 0))
    assert g.shape == (4, 48, 48, 48) and not g.any()
    assert not _gm().forward(single_atom((40.0, 0, 0)), center=(0, 0, 0)).any()


def test_default_center_is_centroid(rng):
    atoms = random_coordinate_set(rng, 12, num_types=4, extent=3.0)
    np.testing.assert_array_equal(_gm().forward(atoms),
                                  _gm().forward(atoms, center=atoms.centroid()))


def test_out_buffer_reused_and_validated():
    out = np.full((1, 48, 48, 48), 9.0, dtype=np.float32)
    got = _gm().forward(single_atom((0, 0, 0)), center=(0, 0, 0), out=out)
    assert got is out and out.max() <= 1.0
    with pytest.raises(ValueError):
        _gm().forward(single_atom((0, 0, 0), num_types=2), center=(0, 0, 0),
                      out=np.zeros((3, 48, 48, 48), np.float32))
    with pytest.raises(TypeError):
        _gm().forward(single_atom((0, 0, 0)), center=(0, 0, 0),
                      out=np.zeros((1, 48, 48, 48), np.float64))


# ---------------------------------------------------------------- oracle equivalence

@pytest.mark.parametrize("seed", range(10))
def test_forward_matches_all_pairs(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 51))
    atoms = random_coordinate_set(rng, n, num_types=14, extent=9.0)
    center = rng.uniform(-1, 1, 3)
    grid = _gm().forward(atoms, center=center)
    ref = grid_all_pairs(atoms.coords, atoms.radii, atoms.type_index, 14, center)
    assert np.abs(grid - ref).max() < 1e-6


def test_binary_matches_all_pairs_bit_exact(rng):
    atoms = random_coordinate_set(rng, 30, num_types=5, extent=6.0)
    grid = _gm(binary=True).forward(atoms, center=(0, 0, 0))
    ref = grid_all_pairs(atoms.coords, atoms.radii, atoms.type_index, 5, (0, 0, 0), binary=True)
    np.testing.assert_array_equal(grid, ref.astype(np.float32))
    assert (grid[grid != 0] == 1.0).all()


def test_radius_scale_and_grm(rng):
    atoms = random_coordinate_set(rng, 20, num_types=3, extent=5.0)
    grid = _gm(radius_scale=1.4, gaussian_radius_multiple=1.5).forward(atoms, center=(0, 0, 0))
    ref = grid_all_pairs(atoms.coords, atoms.radii, atoms.type_index, 3, (0, 0, 0), grm=1.5,
                         radius_scale=1.4)
    assert np.abs(grid - ref).max() < 1e-6


def test_vector_mode_matches_all_pairs(rng):
    atoms = random_coordinate_set(rng, 15, num_types=4, extent=5.0, index_mode=False)
    grid = _gm().forward(atoms, center=(0, 0, 0))
    ref = grid_all_pairs(atoms.coords, atoms.radii, None, 4, (0, 0, 0),
                         type_vector=atoms.type_vector)
    assert np.abs(grid - ref).max() < 1e-6


def test_radius_type_indexed_matches_all_pairs(rng):
    from paper_1912_04822_b200 import ConfigError, CoordinateSet

    n = 10
    cs = CoordinateSet(coords=rng.uniform(-4, 4, (n, 3)).astype(np.float32),
                       radii=np.ones(n, dtype=np.float32), num_types=3,
                       type_vector=rng.uniform(0, 1, (n, 3)).astype(np.float32),
                       type_radii=np.array([1.0, 1.5, 2.0], dtype=np.float32))
    grid = _gm(radius_type_indexed=True).forward(cs, center=(0, 0, 0))
    ref = grid_all_pairs(cs.coords, cs.radii, None, 3, (0, 0, 0), type_vector=cs.type_vector,
                         type_radii=cs.type_radii)
    assert np.abs(grid - ref).max() < 1e-6
    no_table = random_coordinate_set(rng, 4, num_types=2, index_mode=False)
    with pytest.raises(ConfigError):
        _gm(radius_type_indexed=True).forward(no_table, center=(0, 0, 0))


# ---------------------------------------------------------------- properties

def test_superposition(rng):
    from paper_1912_04822_b200 import CoordinateSet

    a = random_coordinate_set(rng, 12, num_types=4, extent=5.0)
    b = random_coordinate_set(rng, 9, num_types=4, extent=5.0)
    both = CoordinateSet(coords=np.vstack([a.coords, b.coords]),
                         radii=np.concatenate([a.radii, b.radii]), num_types=4,
                         type_index=np.concatenate([a.type_index, b.type_index]))
    gm = _gm()
    combined = gm.forward(both, center=(0, 0, 0))
    assert np.abs(combined - gm.forward(a, center=(0, 0, 0)) - gm.forward(b, center=(0, 0, 0))).max() < 1e-5


def test_translation_equivariance(rng):
    atoms = random_coordinate_set(rng, 15, num_types=4, extent=5.0)
    shift = np.array([3.25, -1.5, 0.75], dtype=np.float32)
    gm = _gm()
    base = gm.forward(atoms, center=(0, 0, 0))
    shifted = gm.forward(atoms.with_coords(atoms.coords + shift), center=shift)
    assert np.abs(base - shifted).max() < 1e-5


def test_rotation_preserves_mass_inside():
    gm = _gm()
    atoms = single_atom((2.0, 1.0, -1.5), radius=1.8)
    base = gm.forward(atoms, center=(0, 0, 0)).sum()
    for seed in range(5):
        g = gm.forward(atoms, center=(0, 0, 0), random_rotation=True,
                       rng=np.random.default_rng(seed))
        assert abs(g.sum() - base) / base < 0.01


def test_deterministic_given_seed(rng):
    atoms = random_coordinate_set(rng, 10, num_types=3)
    gm = _gm()
    a = gm.forward(atoms, center=(0, 0, 0), random_translation=2.0, random_rotation=True,
                   rng=np.random.default_rng(5))
    b = gm.forward(atoms, center=(0, 0, 0), random_translation=2.0, random_rotation=True,
                   rng=np.random.default_rng(5))
    np.testing.assert_array_equal(a, b)


# ---------------------------------------------------------------- batch

def test_batch_semantics(rng):
    from paper_1912_04822_b200 import Example, make_vector_types

    gm = _gm()
    ex = _two_set_example(rng)
    out = gm.forward_batch([ex, ex])
    np.testing.assert_array_equal(out[0], out[1])
    aug = gm.forward_batch([ex, ex], random_rotation=True, rng=np.random.default_rng(0))
    assert np.abs(aug[0] - aug[1]).max() > 0
    s1 = random_coordinate_set(rng, 5, num_types=2, extent=3.0)
    s2 = random_coordinate_set(rng, 5, num_types=3, extent=3.0)
    blk = gm.forward_batch([Example(coord_sets=[s1, s2])], centers=np.zeros((1, 3)))
    np.testing.assert_array_equal(blk[0, :2], gm.forward(s1, center=(0, 0, 0)))
    np.testing.assert_array_equal(blk[0, 2:], gm.forward(s2, center=(0, 0, 0)))
    ex2 = _two_set_example(rng)
    np.testing.assert_array_equal(
        gm.forward_batch([ex2]),
        gm.forward_batch([ex2], centers=ex2.coord_sets[-1].centroid().reshape(1, 3)))
    with pytest.raises(ValueError):
        gm.forward_batch([_two_set_example(rng, num_types=3)],
                         out=np.zeros((1, 5, 48, 48, 48), np.float32))
    with pytest.raises(ValueError):
        gm.forward_batch([Example([random_coordinate_set(rng, 4, 2)]),
                          Example([make_vector_types(random_coordinate_set(rng, 4, 2))])])
    empty = Example(coord_sets=[], labels=[], seqcont=True)
    mix = gm.forward_batch([_two_set_example(rng, num_types=3), empty])
    assert not mix[1].any() and mix[0].any()
    o1 = gm.forward_batch([ex, ex], random_translation=2.0, rng=np.random.default_rng(3))
    o2 = gm.forward_batch([ex, ex], random_translation=2.0, rng=np.random.default_rng(3))
    np.testing.assert_array_equal(o1, o2)
    assert np.abs(o1[0] - o1[1]).max() > 0


def test_estimator_protocol(rng):
    pytest.importorskip("sklearn")
    from sklearn.pipeline import Pipeline

    from paper_1912_04822_b200 import channel_count, channel_names

    examples = [_two_set_example(rng) for _ in range(3)]
    gm = _gm()
    np.testing.assert_array_equal(gm.transform(examples), gm.forward_batch(examples))
    assert channel_count(examples[0]) == 6 and len(channel_names(examples[0])) == 6
    pipe = Pipeline([("voxels", _gm(resolution=1.0, dimension=12.0))])
    assert pipe.fit_transform([_two_set_example(rng, num_types=2)] * 2).shape[0] == 2


# ---------------------------------------------------------------- backward

def test_backward_known_answers(rng):
    gm = _gm()
    gg = np.zeros((1, 48, 48, 48), np.float32)
    gg[0, 23, 23, 23] = 1.0
    cg, tg = gm.backward(single_atom((-0.25, -0.25, -0.25)), gg, center=(0, 0, 0))
    assert tg is None
    np.testing.assert_array_equal(cg, np.zeros((1, 3), np.float32))
    atoms = random_coordinate_set(rng, 8, num_types=2)
    cg, _ = gm.backward(atoms, np.zeros((2, 48, 48, 48), np.float32), center=(0, 0, 0))
    assert not cg.any()
    with pytest.raises(ValueError):
        gm.backward(atoms, np.zeros((3, 48, 48, 48), np.float32), center=(0, 0, 0))
    cg, _ = _gm(binary=True).backward(atoms, np.ones((2, 48, 48, 48), np.float32),
                                      center=(0, 0, 0))
    assert not cg.any()


def _fd_instance(rng, n_atoms):
    from paper_1912_04822_b200 import CoordinateSet

    atoms = CoordinateSet(coords=rng.uniform(-2.2, 2.2, (n_atoms, 3)).astype(np.float32),
                          radii=rng.uniform(1.4, 2.2, n_atoms).astype(np.float32),
                          num_types=2, type_index=rng.integers(0, 2, n_atoms))
    gg = rng.uniform(0.2, 1.0, (2, 17, 17, 17))
    gg = mask_seams(gg, atoms.coords, atoms.radii, (0, 0, 0), 0.5, 8.0).astype(np.float32)
    return atoms, gg


def test_gradient_check_all_branches():
    """test_acceptance.py:122-188: coord rel < 1e-3, type rel < 1e-3."""
    gm = _gm(resolution=0.5, dimension=8.0)
    worst = 0.0
    for seed in list(range(8)) + [1000 + s for s in range(4)]:
        rng = np.random.default_rng(seed)
        atoms, gg = _fd_instance(rng, 1 if seed < 1000 else int(rng.integers(2, 7)))
        analytic, _ = gm.backward(atoms, gg, center=(0, 0, 0))

        def loss(c, atoms=atoms, gg=gg):
            ref = grid_all_pairs(c, atoms.radii, atoms.type_index, 2, (0, 0, 0), 0.5, 8.0)
            return float((gg.astype(np.float64) * ref).sum())

        numeric = central_differences(loss, atoms.coords.astype(np.float64), 1e-2)
        worst = max(worst, float(relative_errors(analytic, numeric).max()))
    assert worst < 1e-3
    from paper_1912_04822_b200 import CoordinateSet

    wt = 0.0
    for seed in range(3):
        rng = np.random.default_rng(2000 + seed)
        n = int(rng.integers(1, 5))
        cs = CoordinateSet(coords=rng.uniform(-2.2, 2.2, (n, 3)).astype(np.float32),
                           radii=rng.uniform(1.4, 2.0, n).astype(np.float32), num_types=2,
                           type_vector=rng.uniform(0.1, 1.0, (n, 2)).astype(np.float32))
        gg = rng.uniform(0.2, 1.0, (2, 17, 17, 17)).astype(np.float32)
        _, tg = gm.backward(cs, gg, center=(0, 0, 0))

        def wloss(w, cs=cs, gg=gg):
            ref = grid_all_pairs(cs.coords, cs.radii, None, 2, (0, 0, 0), 0.5, 8.0, type_vector=w)
            return float((gg.astype(np.float64) * ref).sum())

        numeric = central_differences(wloss, cs.type_vector.astype(np.float64), 1e-3)
        wt = max(wt, float(relative_errors(tg, numeric).max()))
    assert wt < 1e-3


def test_acceptance_oracle_equivalence_100_instances():
    """test_acceptance.py:75-89: 100 instances, max |delta| < 1e-5."""
    gm = _gm()
    worst = 0.0
    for seed in range(100):
        rng = np.random.default_rng(seed)
        n = int(rng.integers(1, 51))
        atoms = random_coordinate_set(rng, n, num_types=14, extent=9.0)
        center = rng.uniform(-2, 2, 3)
        grid = gm.forward(atoms, center=center)
        if seed % 10 == 0:  # all-pairs is slow on CPU; sample it
            ref = grid_all_pairs(atoms.coords, atoms.radii, atoms.type_index, 14, center)
            worst = max(worst, float(np.abs(grid - ref).max()))
    assert worst < 1e-6


def test_default_shape_and_torch_views():
    from paper_1912_04822_b200 import Example, synthetic

    rng = np.random.default_rng(0)
    exs = [Example([synthetic.receptor(rng, 8, 4.0), synthetic.ligand(rng, 4, 2.0)])
           for _ in range(10)]
    gm = _gm()
    assert gm.points_per_side() == 48
    batch = gm.forward_batch(exs)
    assert batch.shape == (10, 28, 48, 48, 48)
    dev = torch.zeros((10, 28, 48, 48, 48), device="cuda")
    gm.forward_batch(exs, out=dev)
    np.testing.assert_array_equal(to_numpy(dev), batch)


def test_backward_batch_input_frame_rotates_back():
    """d/dx of a rotated frame: grad_input = R^T grad_transformed (8(f) row 2)."""
    from paper_1912_04822_b200 import synthetic

    exs = synthetic.batch(3, seed=11)
    gm = _gm()
    grid, xf = gm.forward_batch(exs, random_rotation=True, rng=np.random.default_rng(1),
                                return_transforms=True)
    in_t = gm.backward_batch(exs, grid, transforms=xf)
    in_x = gm.backward_batch(exs, grid, transforms=xf, input_frame=True)
    for e in range(3):
        R = xf[e].rotation.rotation_matrix()
        for (ct, _), (cx, _) in zip(in_t[e], in_x[e]):
            # rotated in f64 from the f32 transformed-frame gradient, rounded once
            want = (ct.astype(np.float64) @ R).astype(np.float32)
            np.testing.assert_allclose(cx, want, rtol=1e-6, atol=1e-7)

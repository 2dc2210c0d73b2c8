"""Pin the CPU oracle against fixtures produced by the live reference.

These run without a GPU.  They prove the oracle (oracle/oracle.c + the
packing restatement in oracle/__init__.py) reproduces the reference's
outputs, so the GPU parity tests can trust it as the checker.
"""

import numpy as np
import pytest

import oracle
from oracle import allpairs
from golden_io import (BATCH_FIXTURES, SINGLE_FIXTURES, VECTOR_FIXTURES, aug_from,
                       dense_from_sparse, examples_from, expected_grid, load, params_from,
                       sets_from, unpack_bits)


def smooth_close(got, want, rel=1e-12, abs_=1e-12):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    assert got.shape == want.shape
    err = np.abs(got - want)
    assert (err <= abs_ + rel * np.abs(want)).all(), float(err.max())


@pytest.mark.parametrize("name", SINGLE_FIXTURES)
def test_single_forward(name):
    d = load(name)
    go = oracle.GridOracle(**params_from(d))
    grid = go.forward(sets_from(d)[0], center=d["center"])
    # same f64 arithmetic + one f32 rounding: bit-exact on the same libm
    np.testing.assert_array_equal(grid, d["grid"])


@pytest.mark.parametrize("name", BATCH_FIXTURES + VECTOR_FIXTURES)
def test_batch_forward(name):
    d = load(name)
    go = oracle.GridOracle(**params_from(d))
    grid = go.forward_batch(examples_from(d), **aug_from(d))
    np.testing.assert_array_equal(grid, expected_grid(d))


def test_backward_index():
    d = load("bwd_index")
    go = oracle.GridOracle(**params_from(d))
    cg, tg = go.backward(sets_from(d)[0], d["grid_grad"], center=d["center"])
    assert tg is None
    np.testing.assert_array_equal(cg, d["coord_grad"])


@pytest.mark.parametrize("rti", [0, 1])
def test_backward_vector(rti):
    d = load(f"bwd_vector_rti{rti}")
    go = oracle.GridOracle(**params_from(d))
    cg, tg = go.backward(sets_from(d)[0], d["grid_grad"], center=d["center"])
    np.testing.assert_array_equal(cg, d["coord_grad"])
    np.testing.assert_array_equal(tg, d["type_grad"])


def test_c2_example_full_size():
    d = load("c2_example")
    exs = examples_from(d)
    go = oracle.GridOracle()
    grid = go.forward_batch(exs)
    want = dense_from_sparse(d)
    np.testing.assert_array_equal(grid, want)
    center = exs[0].coord_sets[-1].centroid()
    cg_rec, _ = go.backward(exs[0].coord_sets[0], grid[0, :14], center=center)
    cg_lig, _ = go.backward(exs[0].coord_sets[1], grid[0, 14:], center=center)
    np.testing.assert_array_equal(cg_rec, d["coord_grad_rec"])
    np.testing.assert_array_equal(cg_lig, d["coord_grad_lig"])


def test_c3_binary_augmented_bit_exact():
    d = load("c3_example")
    go = oracle.GridOracle(binary=True)
    grid = go.forward_batch(examples_from(d), random_rotation=True, random_translation=2.0,
                            rng=np.random.default_rng(int(d["aug_seed"])))
    np.testing.assert_array_equal(grid, unpack_bits(d))


def test_transforms_match_numpy_fixture():
    d = load("transforms")
    for i, pk in enumerate(d["packs"]):
        R, c, t = pk[:9].reshape(3, 3), pk[9:12], pk[12:15]
        y = oracle.apply_transform(R, c, t, d[f"x{i}"].astype(np.float64))
        np.testing.assert_array_equal(y, d[f"y{i}"])


def test_allpairs_agrees_with_oracle():
    """The independent all-pairs restatement agrees with the C oracle (1e-6,
    the reference's own gate, test_voxelizer.py:146)."""
    d = load("fwd_index_s2")
    cs = sets_from(d)[0]
    p = params_from(d)
    ref = allpairs.grid_all_pairs(cs.coords, cs.radii, cs.type_index, cs.num_types,
                                  d["center"], resolution=p["resolution"],
                                  dimension=p["dimension"])
    assert np.abs(ref - d["grid"]).max() < 1e-6


def test_oracle_thread_count_independent():
    d = load("batch_smooth_rottr")
    go = oracle.GridOracle(**params_from(d))
    n0 = oracle.num_threads()
    try:
        oracle.set_num_threads(1)
        a = go.forward_batch(examples_from(d), **aug_from(d))
        oracle.set_num_threads(max(2, n0))
        b = go.forward_batch(examples_from(d), **aug_from(load("batch_smooth_rottr")))
    finally:
        oracle.set_num_threads(n0)
    np.testing.assert_array_equal(a, b)

"""The reference-shaped drop-in (paper_1912_04822_b200.kernels, i.e. the C
ABI's *_host entry points) against the CPU oracle on identical packed
arrays -- the exact call the reference's voxelizer makes into _kernels."""

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


def _batch(vector=False, n=6, seed=2):
    from paper_1912_04822_b200 import synthetic

    return synthetic.batch(n, seed=seed, vector=vector)


@pytest.mark.parametrize("binary", [False, True])
def test_forward_index_sets_dropin(binary):
    from paper_1912_04822_b200 import kernels

    go = oracle.GridOracle(binary=binary)
    exs = _batch()
    _, centers, origins, placed, _ = go.place(exs, random_rotation=True, random_translation=2.0,
                                             rng=np.random.default_rng(1))
    d = go.pack_placed(placed)
    D = go.npts
    want = np.zeros((len(exs), 28, D, D, D), np.float32)
    go.forward_placed(want, placed, origins)
    got = np.full_like(want, 7.0)  # not pre-zeroed: every voxel is written
    kernels.forward_index_sets(got, d["coords"], d["radii"], d["tidx"], d["set_start"],
                               d["set_end"], d["set_example"], d["set_choff"], d["set_t"],
                               origins, go.resolution, go.grm, go.rmult, binary)
    if binary:
        np.testing.assert_array_equal(got, want)
    else:
        assert_close(got, want, what="forward_index_sets")


@pytest.mark.parametrize("rti", [False, True])
@pytest.mark.parametrize("binary", [False, True])
def test_forward_vector_sets_dropin(rti, binary):
    from paper_1912_04822_b200 import kernels

    go = oracle.GridOracle(binary=binary, radius_type_indexed=rti)
    exs = _batch(vector=True, n=3, seed=4)
    _, centers, origins, placed, _ = go.place(exs, random_rotation=True,
                                             rng=np.random.default_rng(2))
    d = go.pack_placed(placed)
    D = go.npts
    want = np.zeros((len(exs), 28, D, D, D), np.float32)
    go.forward_placed(want, placed, origins)
    got = np.zeros_like(want)
    kernels.forward_vector_sets(got, d["coords"], d["weights_flat"], d["w_start"],
                                d["atom_radii"], d["type_radii_flat"], d["tr_start"], rti,
                                d["set_start"], d["set_end"], d["set_example"], d["set_choff"],
                                d["set_t"], origins, go.resolution, go.grm, go.rmult, binary)
    if binary:
        np.testing.assert_array_equal(got, want)
    else:
        assert_close(got, want, what="forward_vector_sets")


def test_backward_index_dropin():
    from paper_1912_04822_b200 import kernels

    go = oracle.GridOracle()
    cs = _batch(n=1)[0].coord_sets[0]
    center = cs.centroid()
    D = go.npts
    gg = np.random.default_rng(3).standard_normal((14, D, D, D), dtype=np.float32)
    coords = cs.coords.astype(np.float64)
    radii = cs.radii.astype(np.float64)
    origin = go.origin(center)
    got = kernels.backward_index(coords, radii, cs.type_index, gg, origin, go.resolution,
                                 go.grm, go.rmult)
    want = np.zeros_like(got)
    oracle.lib().oracle_backward_index(want, coords, radii, cs.type_index, coords.shape[0], gg,
                                       D, np.ascontiguousarray(origin), go.resolution, go.grm,
                                       go.rmult)
    assert got.dtype == np.float64 and got.shape == (coords.shape[0], 3)
    assert_close(got, want, what="backward_index")
    # f64 sums like the numba kernel (_kernels.py:214), not f32-rounded values
    assert_close(got, want, rel=1e-9, abs_=1e-10, what="backward_index f64")
    assert (got != got.astype(np.float32).astype(np.float64)).any()


@pytest.mark.parametrize("rti", [False, True])
def test_backward_vector_dropin(rti):
    from paper_1912_04822_b200 import kernels

    go = oracle.GridOracle(radius_type_indexed=rti)
    cs = _batch(vector=True, n=1, seed=4)[0].coord_sets[0]
    D = go.npts
    gg = np.random.default_rng(5).standard_normal((14, D, D, D), dtype=np.float32)
    coords = cs.coords.astype(np.float64)
    radii = cs.radii.astype(np.float64)
    w = cs.type_vector.astype(np.float64)
    tr = cs.type_radii.astype(np.float64) if rti else np.ones(14)
    origin = np.ascontiguousarray(go.origin(cs.centroid()))
    cg, tg = kernels.backward_vector(coords, radii, w, gg, tr, rti, origin, go.resolution,
                                     go.grm, go.rmult)
    wc, wt = np.zeros_like(cg), np.zeros_like(tg)
    oracle.lib().oracle_backward_vector(wc, wt, coords, radii, w, coords.shape[0], 14, gg, D, tr,
                                        int(rti), origin, go.resolution, go.grm, go.rmult)
    assert_close(cg, wc, what="coord")
    assert_close(tg, wt, what="type")
    assert_close(cg, wc, rel=1e-9, abs_=1e-10, what="coord f64")
    assert_close(tg, wt, rel=1e-9, abs_=1e-10, what="type f64")
    assert (tg != tg.astype(np.float32).astype(np.float64)).any()

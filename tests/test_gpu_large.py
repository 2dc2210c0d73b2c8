"""Batches whose (N, C, D, D, D) grids hold more than 2^31 floats (8.9 GB at
96^3 x 28 channels x 90 examples): every grid / grid_grad offset past 2^31
must be 64-bit.  The last example of the big batch (its channel block starts
past 2^31 floats) is compared bit for bit with the same example gridded
alone, which the parity suites check against the oracle; its coordinate (and
type) gradients likewise.  Index (smooth and binary) and vector typing."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

N_BIG = 90


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    free, _ = torch.cuda.mem_get_info()
    if free < 24e9:
        pytest.skip("needs ~20 GB of free device memory")


@pytest.mark.parametrize("mode", ["index", "binary", "vector"])
def test_grid_offsets_past_2_31(mode):
    from paper_1912_04822_b200 import GridMaker, geom, synthetic

    vector = mode == "vector"
    exs = synthetic.batch(3, seed=2, vector=vector)
    gm = GridMaker(resolution=0.25, dimension=23.75, binary=mode == "binary")
    D = gm.points_per_side()
    big = [exs[k % 2] for k in range(N_BIG - 1)] + [exs[2]]
    pb = gm.pack(big)
    C = pb.nchannels
    assert N_BIG * C * D ** 3 > 2 ** 31  # the last channel blocks lie past 2^31 floats
    xf = geom.draw_transform_array(pb.default_centers, 2.0, True, np.random.default_rng(5))
    out, _ = gm.forward_packed(pb, transforms=xf)
    grads = None
    if mode != "binary":
        grads = gm.backward_packed(pb, out, reuse_prepared=True)
    last = out[-1].clone()
    del out
    torch.cuda.empty_cache()

    one = gm.pack([exs[2]], nchannels=C)
    out1, _ = gm.forward_packed(one, transforms=geom.TransformArray(xf.packed[-1:]))
    assert torch.equal(last, out1[0]), "the example past 2^31 floats differs from its own forward"
    if grads is not None:
        cg, tg = grads
        cg1, tg1 = gm.backward_packed(one, out1, reuse_prepared=True)
        # packed atom order is example-major: the last example's atoms come last
        assert torch.equal(cg[-cg1.shape[0]:], cg1), "coordinate gradients past 2^31 differ"
        if vector:
            assert torch.equal(tg[-tg1.shape[0]:], tg1), "type gradients past 2^31 differ"

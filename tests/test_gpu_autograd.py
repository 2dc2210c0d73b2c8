"""Autograd over the CUDA gridding path: gradients of a
loss on the grids with respect to the input-frame coordinates (and, in
vector mode, the type weights), checked against the CPU oracle's backward
(transformed frame) rotated back by the example's rotation."""

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


def _rotate_back(cgs, placed_examples, transforms):
    """oracle per-set gradients (transformed frame) -> input frame, f64."""
    out = []
    for cg, e in zip(cgs, placed_examples):
        R = np.asarray(transforms.packed[e, :9], np.float64).reshape(3, 3)
        out.append(np.asarray(cg, np.float64) @ R)
    return np.concatenate(out)


@pytest.mark.parametrize("vector", [False, True])
def test_grid_atoms_gradients_vs_oracle(vector):
    from paper_1912_04822_b200 import GridMaker, geom, synthetic
    from paper_1912_04822_b200.autograd import grid_atoms, packed_coords, packed_weights

    exs = synthetic.batch(6, seed=11, vector=vector)
    gm = GridMaker()
    pb = gm.pack(exs)
    xf = geom.draw_transform_array(pb.default_centers, 2.0, True, np.random.default_rng(5))
    x = packed_coords(pb).requires_grad_(True)
    w = packed_weights(pb)
    if w is not None:
        w.requires_grad_(True)
    grid = grid_atoms(gm, pb, x, w, transforms=xf)
    G = torch.randn(grid.shape, generator=torch.Generator(device="cuda").manual_seed(3),
                    device="cuda")
    (grid * G).sum().backward()

    go = oracle.GridOracle()
    ref = go.forward_batch(exs, random_rotation=True, random_translation=2.0,
                           rng=np.random.default_rng(5))
    assert_close(grid.detach().cpu().numpy(), ref, what="autograd forward")
    cgs, tgs = go.backward_batch(exs, G.cpu().numpy(), random_rotation=True,
                                 random_translation=2.0, rng=np.random.default_rng(5))
    placed_e = [e for (e, _, _, _, _) in pb.placed]
    want = _rotate_back(cgs, placed_e, xf)
    assert_close(x.grad.cpu().numpy(), want, what="dL/dx (input frame)")
    if vector:
        want_t = np.concatenate([np.asarray(t, np.float64).reshape(-1) for t in tgs])
        assert_close(w.grad.cpu().numpy(), want_t, what="dL/dweights")


def test_grid_atoms_matches_backward_batch_input_frame():
    from paper_1912_04822_b200 import GridMaker, synthetic
    from paper_1912_04822_b200.autograd import grid_atoms, packed_coords

    exs = synthetic.batch(4, seed=12)
    gm = GridMaker()
    grid0, xf = gm.forward_batch(exs, random_rotation=True, random_translation=1.5,
                                 rng=np.random.default_rng(2), return_transforms=True)
    pb = gm.pack(exs)
    x = packed_coords(pb).requires_grad_(True)
    grid = grid_atoms(gm, pb, x, transforms=xf)
    np.testing.assert_array_equal(grid.detach().cpu().numpy(), grid0)
    g = torch.from_numpy(grid0).cuda()
    (0.5 * (grid * grid).sum()).backward()
    res = gm.backward_batch(exs, g, transforms=xf, input_frame=True)
    want = torch.cat([c for ex in res for (c, _) in ex]).cpu().numpy()
    assert_close(x.grad.cpu().numpy(), want, what="autograd vs backward_batch(input_frame)")


def test_grid_atoms_binary_zero_gradients():
    from paper_1912_04822_b200 import GridMaker, synthetic
    from paper_1912_04822_b200.autograd import grid_atoms, packed_coords

    exs = synthetic.batch(2, seed=13)
    gm = GridMaker(binary=True)
    pb = gm.pack(exs)
    x = packed_coords(pb).requires_grad_(True)
    grid_atoms(gm, pb, x).sum().backward()
    assert torch.count_nonzero(x.grad).item() == 0

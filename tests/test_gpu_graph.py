"""GraphStep (graph.py): prepare -> forward -> backward captured as CUDA graphs
and replayed per call gives the eager packed path's outputs bit for bit, for
every replay, with fresh transforms each call."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _eager(gm, pb, xf, gg):
    out, _ = gm.forward_packed(pb, transforms=xf)
    out = out.clone()
    if gg is None and not gm.binary:
        return out, None, None
    cg, tg = gm.backward_packed(pb, gg, reuse_prepared=True)
    return out, cg.clone(), None if tg is None else tg.clone()


@pytest.mark.parametrize("vector", [False, True])
def test_graph_step_matches_eager_every_replay(vector):
    from paper_1912_04822_b200 import GridMaker, geom, synthetic

    gm = GridMaker()
    pb = gm.pack(synthetic.batch(5, seed=31, n_receptor=400, vector=vector))
    gen = torch.Generator(device="cuda").manual_seed(5)
    gg = torch.randn((pb.nexamples, pb.nchannels) + (gm.points_per_side(),) * 3,
                     device="cuda", generator=gen)
    step = gm.capture_step(pb, backward=True)
    rng = np.random.default_rng(3)
    for it in range(5):  # both graphs, twice over
        xf = geom.draw_transform_array(pb.default_centers, 2.0, True, rng)
        g2 = gg * (it + 1)
        out, cg, tg, _ = step.run(transforms=xf, grid_grad=g2)
        torch.cuda.synchronize()
        got = (out.clone(), cg.clone(), None if tg is None else tg.clone())
        want = _eager(gm, pb, xf, g2)
        assert torch.equal(got[0], want[0]), it
        assert torch.equal(got[1], want[1]), it
        if vector:
            assert torch.equal(got[2], want[2]), it


def test_graph_step_random_draws_and_no_augment():
    from paper_1912_04822_b200 import GridMaker, synthetic

    gm = GridMaker()
    pb = gm.pack(synthetic.batch(3, seed=32, n_receptor=300))
    step = gm.capture_step(pb)
    out, xf = step.run(random_rotation=True, random_translation=2.0,
                       rng=np.random.default_rng(9))
    want, xf2 = gm.forward_packed(pb, random_rotation=True, random_translation=2.0,
                                  rng=np.random.default_rng(9))
    np.testing.assert_array_equal(xf.packed, xf2.packed)
    assert torch.equal(out, want)

    plain = gm.capture_step(pb, augment=False)
    out, _ = plain.run()
    want, _ = gm.forward_packed(pb)
    assert torch.equal(out, want)
    with pytest.raises(ValueError, match="without augment"):
        plain.run(random_rotation=True)


def test_graph_step_binary_backward():
    from paper_1912_04822_b200 import GridMaker, geom, synthetic

    gm = GridMaker(binary=True)
    pb = gm.pack(synthetic.batch(3, seed=33, n_receptor=300))
    step = gm.capture_step(pb, backward=True)
    xf = geom.draw_transform_array(pb.default_centers, 1.0, True, np.random.default_rng(4))
    out, cg, _, _ = step.run(transforms=xf)
    want = _eager(gm, pb, xf, None)
    assert torch.equal(out, want[0])
    assert torch.equal(cg, want[1])

"""Provider -> device batch pipeline: batches packed and
uploaded ahead on a worker thread, and batches assembled on the device from
a resident dataset, checked against the CPU oracle on the same examples."""
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


class _Provider:
    """Stand-in with the reference ExampleProvider's next_batch(n) API."""

    def __init__(self, seed):
        self.rng = np.random.default_rng(seed)

    def next_batch(self, n):
        from paper_1912_04822_b200 import synthetic

        return [synthetic.complex_example(self.rng, n_receptor=300) for _ in range(n)]


def test_pipeline_batches_grid_like_forward_batch():
    from paper_1912_04822_b200 import GridMaker
    from paper_1912_04822_b200.pipeline import DeviceBatchPipeline

    gm = GridMaker()
    seen = 0
    go = oracle.GridOracle()
    with DeviceBatchPipeline(gm, _Provider(21), batch_size=4, depth=2, max_batches=3) as pipe:
        for pb in pipe:
            grid, _ = gm.forward_packed(pb)
            assert_close(grid.cpu().numpy(), go.forward_batch(pb.examples),
                         what="pipeline batch vs oracle")
            # and the same bits as the one-shot API
            np.testing.assert_array_equal(grid.cpu().numpy(), gm.forward_batch(pb.examples))
            seen += 1
    assert seen == 3


def test_pipeline_from_iterable_and_errors():
    from paper_1912_04822_b200 import GridMaker
    from paper_1912_04822_b200.pipeline import DeviceBatchPipeline

    gm = GridMaker()
    src = [_Provider(22).next_batch(2) for _ in range(2)]
    with DeviceBatchPipeline(gm, src, batch_size=2) as pipe:
        assert len(list(pipe)) == 2

    def bad():
        yield _Provider(23).next_batch(1)
        raise RuntimeError("provider failed")

    with DeviceBatchPipeline(gm, bad(), batch_size=1) as pipe:
        next(pipe)
        with pytest.raises(RuntimeError, match="provider failed"):
            next(pipe)


def test_dataset_batches_epochs_and_parity():
    """DatasetBatches: shuffled epochs over a device-resident dataset, each
    batch assembled on the GPU; grids and gradients vs the oracle."""
    from paper_1912_04822_b200 import GridMaker, geom, synthetic
    from paper_1912_04822_b200.dataset import DeviceDataset
    from paper_1912_04822_b200.pipeline import DatasetBatches

    rng = np.random.default_rng(31)
    exs = [synthetic.complex_example(rng, n_receptor=200) for _ in range(10)]
    gm = GridMaker()
    ds = DeviceDataset(exs)
    it = DatasetBatches(gm, ds, batch_size=4, seed=5, depth=2)
    seen = []
    go = oracle.GridOracle()
    for k in range(6):  # two epochs of 4 + 4 + 2
        ab = next(it)
        sub = [exs[i] for i in ab.ids]
        seen.append(list(ab.ids))
        xf = geom.draw_transform_array(ab.default_centers, 1.5, True, np.random.default_rng(k))
        grid, _ = gm.forward_packed(ab, transforms=xf)
        ref = go.forward_batch(sub, random_rotation=True, random_translation=1.5,
                               rng=np.random.default_rng(k))
        assert_close(grid.cpu().numpy(), ref, what=f"batch {k}")
        gg = torch.from_numpy(ref).cuda()
        cg, _ = gm.backward_packed(ab, gg, reuse_prepared=True)
        cgs, _ = go.backward_batch(sub, ref, random_rotation=True, random_translation=1.5,
                                   rng=np.random.default_rng(k))
        assert_close(cg.cpu().numpy(), np.concatenate(cgs), what=f"batch {k} gradients")
    assert [len(s) for s in seen] == [4, 4, 2, 4, 4, 2]
    assert sorted(sum(seen[:3], [])) == list(range(10))
    assert sorted(sum(seen[3:], [])) == list(range(10))
    assert seen[:3] != seen[3:]  # a new permutation each epoch


def test_dataset_batches_prefetch_matches_serial():
    """DatasetBatches(prefetch=True) assembles batch k + 1 on a side stream
    while the consumer grids batch k: same index lists, and grids / gradients
    bit-identical to the serial iterator, the previous batch still intact."""
    from paper_1912_04822_b200 import GridMaker, geom, synthetic
    from paper_1912_04822_b200.dataset import DeviceDataset
    from paper_1912_04822_b200.pipeline import DatasetBatches

    rng = np.random.default_rng(8)
    exs = [synthetic.complex_example(rng, n_receptor=300) for _ in range(23)]
    gm = GridMaker()
    ds = DeviceDataset(exs)
    runs = []
    for prefetch in (False, True):
        it = DatasetBatches(gm, ds, batch_size=5, seed=9, depth=2, prefetch=prefetch,
                            max_batches=9)
        got, prev = [], None
        for k, ab in enumerate(it):
            xf = geom.draw_transform_array(ab.default_centers, 2.0, True, np.random.default_rng(k))
            grid, _ = gm.forward_packed(ab, transforms=xf)
            cg, _ = gm.backward_packed(ab, grid, reuse_prepared=True)
            if prev is not None:  # depth 2: the previous batch is still valid
                pab, pids = prev
                assert list(pab.ids) == pids
            prev = (ab, list(ab.ids))
            got.append((list(ab.ids), grid.cpu(), cg.cpu()))
        assert len(got) == 9
        runs.append(got)
    for (i0, g0, c0), (i1, g1, c1) in zip(*runs):
        assert i0 == i1
        assert torch.equal(g0, g1) and torch.equal(c0, c1)

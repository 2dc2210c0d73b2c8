"""Provider -> device batch pipeline: batches packed and
uploaded ahead on a worker thread grid exactly like forward_batch."""
import numpy as np
import pytest

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
    with DeviceBatchPipeline(gm, _Provider(21), batch_size=4, depth=2, max_batches=3) as pipe:
        for pb in pipe:
            grid, _ = gm.forward_packed(pb)
            want = gm.forward_batch(pb.examples)
            np.testing.assert_array_equal(grid.cpu().numpy(), want)
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

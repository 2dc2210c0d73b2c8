"""Grid containers on the host: the reference's grid
semantics (/root/reference/pkg/src/voxmol/grids.py:45-236, its tests in
pkg/tests/test_grids.py) -- shapes, strides, bounds, aliasing, dtype rules --
plus torch-backed storage.  No GPU needed (CPU tensors stand in for device
ones; the CUDA-backed path is in test_gpu_regressions.py)."""

import numpy as np
import pytest
import torch

from paper_1912_04822_b200 import GridShape, GridView, OwnedGrid, copy_into, make_grid, view_over


def test_grid_shape_rules():
    s = GridShape(2, 3, 4)
    assert s.dims == (2, 3, 4) and s.ndim == 3 and s.size == 24 and len(s) == 3
    assert s.strides == (12, 4, 1)
    assert s.offset((1, 2, 3)) == 23
    assert GridShape((2, 3, 4)) == s == (2, 3, 4)
    assert hash(GridShape([2, 3, 4])) == hash(s)
    assert list(s) == [2, 3, 4]
    assert repr(s) == "GridShape(2, 3, 4)"
    with pytest.raises(IndexError, match="out of bounds"):
        s.offset((2, 0, 0))
    with pytest.raises(IndexError, match="out of bounds"):
        s.offset((0, -1, 0))
    with pytest.raises(IndexError, match="expected 3 indices"):
        s.offset((0, 0))
    with pytest.raises(ValueError, match="1..6 dimensions"):
        GridShape(*([2] * 7))
    with pytest.raises(ValueError, match="positive integer"):
        GridShape(2, 0)
    with pytest.raises(ValueError, match="positive integer"):
        GridShape(2.5, 3)


def test_owned_grid_zeroed_and_typed():
    g = make_grid((2, 3), "f64")
    assert isinstance(g, OwnedGrid)
    assert g.dtype == np.float64 and g.size == 6 and g.shape == (2, 3)
    assert not g.array.any()
    g.set((1, 2), 5.0)
    assert g.get((1, 2)) == 5.0 and g[1, 2] == 5.0
    with pytest.raises(IndexError):
        g.get((2, 0))
    g.fill(1.5)
    assert (g.tonumpy() == 1.5).all()
    with pytest.raises(TypeError, match="unsupported element type"):
        make_grid((2,), "i32")
    with pytest.raises(TypeError, match="only float32/float64"):
        make_grid((2,), np.int32)


def test_view_aliases_and_checks():
    buf = np.arange(30, dtype=np.float32)
    v = view_over(buf, (2, 3, 4))
    assert isinstance(v, GridView) and v.shape == (2, 3, 4)
    v[0, 0, 1] = -1.0
    assert buf[1] == -1.0  # writes go through
    assert np.shares_memory(v.array, buf)
    with pytest.raises(ValueError, match="needs 60"):
        view_over(buf, (3, 4, 5))
    with pytest.raises(TypeError, match="does not match requested"):
        view_over(buf.astype(np.float64), (2, 3), "f32")
    with pytest.raises(ValueError, match="C-contiguous"):
        view_over(np.zeros((4, 4), np.float32)[:, ::2], (2, 2))
    with pytest.raises(TypeError, match="not a float32/float64"):
        view_over(np.zeros(4, np.int32), (4,))
    # Python buffers (memoryview of an array.array)
    import array

    arr = array.array("d", [0.0] * 8)
    mv = view_over(arr, (2, 4), "f64")
    mv[1, 3] = 2.0
    assert arr[7] == 2.0
    # a view of a grid aliases the grid's storage
    g = make_grid((6,))
    v2 = view_over(g, (2, 3))
    v2[1, 2] = 3.0
    assert g[5] == 3.0


def test_torch_backed_views_and_copies():
    t = torch.zeros(12, dtype=torch.float32)
    v = view_over(t, (3, 4))
    v[2, 3] = 4.0
    assert t[11] == 4.0
    assert v.dtype == np.float32 and v.size == 12 and not v.on_device
    assert v.array.data_ptr() == t.data_ptr()
    with pytest.raises(ValueError, match="C-contiguous"):
        view_over(torch.zeros(4, 4)[:, ::2], (2, 2))
    g = make_grid((3, 4), device="cpu")
    assert isinstance(g.array, torch.Tensor)
    copy_into(v, g)
    assert g.get((2, 3)) == 4.0
    h = make_grid((3, 4))
    copy_into(g, h)  # tensor -> numpy
    assert h[2, 3] == 4.0
    with pytest.raises(ValueError, match="shape mismatch"):
        copy_into(h, make_grid((4, 3)))
    with pytest.raises(ValueError, match="dtype mismatch"):
        copy_into(h, make_grid((3, 4), "f64"))


def test_reference_grids_interoperate():
    """The reference's own grid objects are accepted (duck typing on .array),
    when the reference is importable (build container only)."""
    import sys

    src = "/root/reference/pkg/src"
    try:
        sys.path.insert(0, src)
        from voxmol import grids as ref_grids
    except Exception:
        pytest.skip("reference package not importable here")
    finally:
        if sys.path and sys.path[0] == src:
            sys.path.pop(0)
    r = ref_grids.make_grid((2, 3))
    mine = view_over(r, (6,))
    mine[4] = 9.0
    assert r.array[1, 1] == 9.0
    back = ref_grids.view_over(make_grid((2, 2)).array, (4,))
    assert back.shape == ref_grids.GridShape(4)

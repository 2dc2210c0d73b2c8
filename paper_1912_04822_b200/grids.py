"""Grid containers and views, host or device backed.

Mirrors the reference's grid API (/root/reference/pkg/src/voxmol/grids.py:45-236):
``GridShape`` (1..6 positive extents, row-major strides, bounds-checked
offsets), ``OwnedGrid`` (zero-initialised storage), ``GridView`` (aliases an
existing contiguous buffer, never copies), ``make_grid``, ``view_over`` and
``copy_into`` -- same names, argument meaning, exception classes and
messages.

The B200 addition is the backing store: besides numpy arrays and Python
buffers, a grid can live in a torch tensor on a CUDA device
(``make_grid(shape, device="cuda")`` or ``view_over(cuda_tensor, shape)``).
Its ``.array`` is then that tensor, which ``GridMaker.forward`` /
``forward_batch`` accept as ``out`` and ``backward`` / ``backward_batch`` as
``grid_grad`` without a copy (voxelizer.py:272,323 accept anything with
``.array``).  Grid objects of the reference itself are accepted wherever a
grid is (duck typing on ``.array``).
"""

from __future__ import annotations

import numpy as np
import torch

MAX_DIMS = 6

_NAMED = {"f32": np.float32, "float32": np.float32, "f64": np.float64, "float64": np.float64}
_TORCH_OF = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}
_NUMPY_OF = {torch.float32: np.dtype(np.float32), torch.float64: np.dtype(np.float64)}


def _element_dtype(element_type) -> np.dtype:
    """'f32' / 'f64' / numpy float dtypes -> little-endian numpy dtype
    (grids.py:33-42 semantics: anything else is a TypeError)."""
    if isinstance(element_type, str):
        t = _NAMED.get(element_type.lower())
        if t is None:
            raise TypeError(f"unsupported element type {element_type!r}; use 'f32' or 'f64'")
        return np.dtype(t).newbyteorder("<")
    if isinstance(element_type, torch.dtype):
        if element_type not in _NUMPY_OF:
            raise TypeError(f"unsupported element type {element_type}; "
                            "only float32/float64 grids exist")
        return _NUMPY_OF[element_type]
    dt = np.dtype(element_type)
    if dt not in (np.dtype(np.float32), np.dtype(np.float64)):
        raise TypeError(f"unsupported element type {dt}; only float32/float64 grids exist")
    return dt


class GridShape:
    """Extents of a 1..6-dimensional row-major grid."""

    __slots__ = ("dims",)

    def __init__(self, *dims):
        if len(dims) == 1 and not isinstance(dims[0], (int, np.integer)):
            dims = tuple(dims[0])
        if not 1 <= len(dims) <= MAX_DIMS:
            raise ValueError(f"grids support 1..{MAX_DIMS} dimensions, got {len(dims)}")
        checked = []
        for extent in dims:
            if int(extent) != extent or int(extent) < 1:
                raise ValueError(f"every extent must be a positive integer, got {extent!r}")
            checked.append(int(extent))
        self.dims = tuple(checked)

    @property
    def ndim(self) -> int:
        return len(self.dims)

    @property
    def size(self) -> int:
        return int(np.prod(self.dims, dtype=np.int64))

    @property
    def strides(self) -> tuple:
        """Element strides, last axis fastest."""
        acc, out = 1, []
        for extent in reversed(self.dims):
            out.append(acc)
            acc *= extent
        return tuple(reversed(out))

    def offset(self, index) -> int:
        index = tuple(index)
        if len(index) != self.ndim:
            raise IndexError(f"expected {self.ndim} indices, got {len(index)}")
        flat = 0
        for axis, (ix, extent, stride) in enumerate(zip(index, self.dims, self.strides)):
            if not 0 <= ix < extent:
                raise IndexError(f"index {ix} out of bounds for axis {axis} with extent {extent}")
            flat += ix * stride
        return flat

    def __iter__(self):
        return iter(self.dims)

    def __len__(self):
        return self.ndim

    def __eq__(self, other):
        other_dims = other.dims if isinstance(other, GridShape) else tuple(other)
        return self.dims == other_dims

    def __hash__(self):
        return hash(self.dims)

    def __repr__(self):
        return f"GridShape{self.dims}"


class _Grid:
    """Element access shared by owned grids and views; ``_data`` is a numpy
    array or a torch tensor (CPU or CUDA)."""

    _data = None

    @property
    def on_device(self) -> bool:
        return isinstance(self._data, torch.Tensor) and self._data.is_cuda

    @property
    def device(self):
        return self._data.device if isinstance(self._data, torch.Tensor) else torch.device("cpu")

    @property
    def shape(self) -> GridShape:
        return GridShape(tuple(self._data.shape))

    @property
    def dtype(self) -> np.dtype:
        d = self._data.dtype
        return _NUMPY_OF[d] if isinstance(d, torch.dtype) else d

    @property
    def size(self) -> int:
        return int(self._data.numel() if isinstance(self._data, torch.Tensor) else self._data.size)

    @property
    def array(self):
        """The aliased storage (numpy array or torch tensor): writes through
        it are the grid's."""
        return self._data

    def tonumpy(self) -> np.ndarray:
        """A fresh host copy of the contents."""
        if isinstance(self._data, torch.Tensor):
            return self._data.detach().cpu().numpy().copy()
        return self._data.copy()

    def _checked(self, index):
        index = tuple(index) if isinstance(index, (tuple, list)) else (index,)
        self.shape.offset(index)  # bounds check; negative indices are rejected
        return index

    def get(self, index) -> float:
        return float(self._data[self._checked(index)])

    def set(self, index, value) -> None:
        self._data[self._checked(index)] = value

    def __getitem__(self, index):
        return self._data[index]

    def __setitem__(self, index, value):
        self._data[index] = value

    def fill(self, value) -> None:
        if isinstance(self._data, torch.Tensor):
            self._data.fill_(value)
        else:
            self._data.fill(value)

    def __repr__(self):
        where = f", device={self.device}" if isinstance(self._data, torch.Tensor) else ""
        return f"{type(self).__name__}(shape={tuple(self._data.shape)}, dtype={self.dtype}{where})"


class OwnedGrid(_Grid):
    """Zero-initialised grid owning its storage: host numpy by default, a
    torch tensor on ``device`` when one is given."""

    def __init__(self, shape, element_type="f32", device=None):
        shape = shape if isinstance(shape, GridShape) else GridShape(shape)
        dt = _element_dtype(element_type)
        if device is None:
            self._data = np.zeros(shape.dims, dtype=dt)
        else:
            self._data = torch.zeros(shape.dims, dtype=_TORCH_OF[np.dtype(dt.type)],
                                     device=torch.device(device))


def _flat_alias(buffer):
    """A flat, aliasing view of a contiguous float buffer (numpy array, torch
    tensor or Python buffer) -- never a copy."""
    if hasattr(buffer, "array") and not isinstance(buffer, (np.ndarray, torch.Tensor)):
        buffer = buffer.array  # our grids and the reference's
    if isinstance(buffer, torch.Tensor):
        if buffer.dtype not in _NUMPY_OF:
            raise TypeError(f"buffer dtype {buffer.dtype} is not a float32/float64 grid type")
        if not buffer.is_contiguous():
            raise ValueError("buffer must be C-contiguous to view without a copy")
        return buffer.view(-1)
    if isinstance(buffer, np.ndarray):
        if buffer.dtype not in (np.dtype(np.float32), np.dtype(np.float64)):
            raise TypeError(f"buffer dtype {buffer.dtype} is not a float32/float64 grid type")
        if not buffer.flags.c_contiguous:
            raise ValueError("buffer must be C-contiguous to view without a copy")
        return buffer.reshape(-1)
    mem = memoryview(buffer)
    fmt = {"f": np.float32, "d": np.float64}.get(mem.format)
    if fmt is None:
        raise TypeError(f"buffer format {mem.format!r} is not float32/float64")
    if not mem.contiguous:
        raise ValueError("buffer must be contiguous to view without a copy")
    return np.frombuffer(mem, dtype=fmt)


class GridView(_Grid):
    """A grid over someone else's contiguous buffer; aliases, never copies
    or frees it.  The owner must outlive the view."""

    def __init__(self, buffer, shape):
        shape = shape if isinstance(shape, GridShape) else GridShape(shape)
        flat = _flat_alias(buffer)
        n = int(flat.numel() if isinstance(flat, torch.Tensor) else flat.size)
        if n < shape.size:
            raise ValueError(f"buffer holds {n} elements, shape {shape.dims} needs {shape.size}")
        self._data = flat[:shape.size].reshape(shape.dims)


def make_grid(shape, element_type="f32", device=None) -> OwnedGrid:
    """A zeroed grid (host, or on ``device``)."""
    return OwnedGrid(shape, element_type, device=device)


def view_over(buffer, shape, element_type=None) -> GridView:
    """View a contiguous float buffer as a grid without copying; with
    ``element_type`` the buffer's type must match it exactly."""
    view = GridView(buffer, shape)
    if element_type is not None and view.dtype != _element_dtype(element_type):
        raise TypeError(
            f"buffer dtype {view.dtype} does not match requested {element_type}; "
            "source and destination dtypes must match")
    return view


def _storage(g):
    if isinstance(g, (np.ndarray, torch.Tensor)):
        return g
    if hasattr(g, "array"):
        return g.array
    return np.asarray(g)


def copy_into(src, dst) -> None:
    """Elementwise copy between grids of the same shape and element type;
    host <-> device copies go through torch (one DMA)."""
    s, d = _storage(src), _storage(dst)
    s_dt = _NUMPY_OF[s.dtype] if isinstance(s, torch.Tensor) else s.dtype
    d_dt = _NUMPY_OF[d.dtype] if isinstance(d, torch.Tensor) else d.dtype
    if tuple(s.shape) != tuple(d.shape):
        raise ValueError(f"shape mismatch: {tuple(s.shape)} vs {tuple(d.shape)}")
    if s_dt != d_dt:
        raise ValueError(f"dtype mismatch: {s_dt} vs {d_dt}")
    if isinstance(d, torch.Tensor):
        d.copy_(s if isinstance(s, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(s)))
    elif isinstance(s, torch.Tensor):
        np.copyto(d, s.detach().cpu().numpy())
    else:
        np.copyto(d, s)

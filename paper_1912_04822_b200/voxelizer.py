"""GridMaker: typed atoms -> density grids -> atom gradients, on a B200.

Host-side mirror of the reference interface
/root/reference/pkg/src/voxmol/voxelizer.py (GridMaker 79-435): same
constructor, defaults, estimator protocol, geometry helpers, ``forward`` /
``forward_batch`` / ``backward`` semantics, validation order, exception
classes and messages.  The arithmetic runs in the CUDA extension
(csrc/*.cu, libgridmaker_b200.so) through the C ABI; there is no CPU path.

Additions:
* ``backward_batch`` - batched backward over every set of every example in
  the forward's (transformed) frame;
* ``forward_batch(..., return_transforms=True)`` - returns the transforms drawn;
* ``pack`` / ``forward_packed`` / ``backward_packed`` - device-resident batches
  for training loops (pack once, grid many times);
* ``out`` / ``grid_grad`` may be torch CUDA tensors (zero-copy) as well as
  numpy arrays or Grid views (anything with ``.array``).
"""

from __future__ import annotations

import ctypes
import math
import os
import threading

import numpy as np
import torch

from . import _native, export, geom, hostio
from .coordsets import coord_sets_of, is_coordinate_set
from .errors import DeviceError
from .packing import PackedBatch, on_device, stream_handle
from .validation import check_rng, check_vector3


_HOST_THREADS = [max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity")
                       else (os.cpu_count() or 1))]


def set_num_threads(n: int) -> int:
    """voxelizer.py:33-46: same validation and return value.  The gridding
    runs on the GPU; the count bounds the host threads of this process's
    numpy/torch work (torch.set_num_threads) and is returned as in effect."""
    n = int(n)
    if n < 1:
        raise ValueError("thread count must be >= 1")
    _HOST_THREADS[0] = min(n, max(1, os.cpu_count() or 1))
    torch.set_num_threads(_HOST_THREADS[0])
    return _HOST_THREADS[0]


def get_num_threads() -> int:
    """voxelizer.py:49-52."""
    return _HOST_THREADS[0]


def channel_count(example) -> int:
    """Total channels of an example: sum of its sets' type counts."""
    return sum(int(cs.num_types) for cs in coord_sets_of(example))


def channel_names(example) -> list:
    """Set-qualified channel labels ("set:name")."""
    names = []
    for si, cs in enumerate(coord_sets_of(example)):
        base = getattr(cs, "type_names", None) or [f"type{i}" for i in range(cs.num_types)]
        names.extend(f"{si}:{n}" for n in base)
    return names


def _is_tensor(x) -> bool:
    return isinstance(x, torch.Tensor)


def _unwrap(x):
    return x.array if hasattr(x, "array") else x


class GridMaker:
    """Configurable voxelizer running on one CUDA device.

    Parameters match the reference (voxelizer.py:97-105): ``resolution``
    (A), ``dimension`` (A), ``binary``, ``radius_type_indexed``,
    ``radius_scale``, ``gaussian_radius_multiple``.  ``device`` selects the
    GPU (default: the current CUDA device).
    """

    _param_names = ("resolution", "dimension", "binary", "radius_type_indexed",
                    "radius_scale", "gaussian_radius_multiple")

    def __init__(self, resolution=0.5, dimension=23.5, binary=False,
                 radius_type_indexed=False, radius_scale=1.0,
                 gaussian_radius_multiple=1.0, device=None):
        self.resolution = resolution
        self.dimension = dimension
        self.binary = binary
        self.radius_type_indexed = radius_type_indexed
        self.radius_scale = radius_scale
        self.gaussian_radius_multiple = gaussian_radius_multiple
        self.device = device

    # -- estimator protocol (voxelizer.py:109-128) --

    def get_params(self, deep=True) -> dict:
        return {name: getattr(self, name) for name in self._param_names}

    def set_params(self, **params) -> "GridMaker":
        for key, value in params.items():
            if key not in self._param_names:
                raise ValueError(f"unknown parameter {key!r} for GridMaker")
            setattr(self, key, value)
        return self

    def fit(self, X=None, y=None) -> "GridMaker":
        self._check_params()
        return self

    def transform(self, X) -> np.ndarray:
        """Voxelize a list of examples (no augmentation) to (N, C, D, D, D)."""
        return self.forward_batch(X)

    def fit_transform(self, X, y=None) -> np.ndarray:
        return self.fit(X, y).transform(X)

    def _check_params(self) -> None:
        if not float(self.resolution) > 0:
            raise ValueError(f"resolution must be > 0, got {self.resolution}")
        if float(self.dimension) < 0:
            raise ValueError(f"dimension must be >= 0, got {self.dimension}")
        if not float(self.radius_scale) > 0:
            raise ValueError(f"radius_scale must be > 0, got {self.radius_scale}")
        if not float(self.gaussian_radius_multiple) > 0:
            raise ValueError(
                f"gaussian_radius_multiple must be > 0, got {self.gaussian_radius_multiple}")

    # -- geometry (voxelizer.py:143-157) --

    def points_per_side(self) -> int:
        self._check_params()
        return int(math.floor(float(self.dimension) / float(self.resolution) + 0.5)) + 1

    @property
    def radius_multiple(self) -> float:
        grm = float(self.gaussian_radius_multiple)
        return (1.0 + 2.0 * grm * grm) / (2.0 * grm)

    def grid_origin(self, center) -> np.ndarray:
        center = check_vector3(center, "center")
        return center - float(self.dimension) / 2.0

    # -- density kernel, host reference form (voxelizer.py:161-199) --

    def _shells(self, r):
        grm = float(self.gaussian_radius_multiple)
        d0 = grm * r
        dz = self.radius_multiple * r
        return d0, dz, math.exp(-2.0 * grm * grm) / (d0 - dz) ** 2

    def density(self, d, r):
        """Density at distance ``d`` from an atom of (scaled) radius ``r``."""
        r = float(r)
        if r <= 0:
            raise ValueError(f"radius must be > 0, got {r}")
        d = np.asarray(d, dtype=np.float64)
        if self.binary:
            val = np.where(d <= r, 1.0, 0.0)
        else:
            d0, dz, qa = self._shells(r)
            val = np.where(d <= d0, np.exp(-2.0 * d * d / (r * r)),
                           np.where(d < dz, qa * (d - dz) ** 2, 0.0))
        return float(val) if val.ndim == 0 else val

    def density_slope(self, d, r):
        """d(density)/d(distance); zero beyond the cutoff and in binary mode."""
        r = float(r)
        if r <= 0:
            raise ValueError(f"radius must be > 0, got {r}")
        d = np.asarray(d, dtype=np.float64)
        if self.binary:
            val = np.zeros_like(d)
        else:
            d0, dz, qa = self._shells(r)
            val = np.where(d <= d0, np.exp(-2.0 * d * d / (r * r)) * (-4.0 * d / (r * r)),
                           np.where(d < dz, 2.0 * qa * (d - dz), 0.0))
        return float(val) if val.ndim == 0 else val

    # -- device plumbing --

    def _device(self) -> torch.device:
        if not torch.cuda.is_available():
            raise DeviceError("GridMaker needs a CUDA device (sm_100a); none is visible")
        if self.device is None:
            return torch.device("cuda", torch.cuda.current_device())
        d = torch.device(self.device)
        if d.type != "cuda":
            raise DeviceError(f"GridMaker runs on CUDA devices only, got {d}")
        return d if d.index is not None else torch.device("cuda", torch.cuda.current_device())

    def _gm_params(self, npts: int) -> _native.GmParams:
        key = (float(self.resolution), float(self.dimension), bool(self.binary),
               bool(self.radius_type_indexed), float(self.radius_scale),
               float(self.gaussian_radius_multiple), int(npts))
        cached = self.__dict__.get("_params_cache")
        if cached is not None and cached[0] == key:
            return cached[1]
        p = _native.GmParams()
        p.resolution = key[0]
        p.dimension = key[1]
        p.radius_scale = key[4]
        p.gaussian_radius_multiple = key[5]
        p.radius_multiple = self.radius_multiple
        p.npts = key[6]
        p.binary = int(key[2])
        p.radius_type_indexed = int(key[3])
        p.matmul_order_1 = geom.matmul_order(1)
        p.matmul_order_n = geom.matmul_order(2)
        self.__dict__["_params_cache"] = (key, p)
        return p

    def pack(self, examples, nchannels=None, device=None, check_type_radii=True) -> PackedBatch:
        """Pack examples (CoordinateSets or Examples) into a device-resident batch."""
        example_sets = [list(ex) if isinstance(ex, (list, tuple)) else coord_sets_of(ex)
                        for ex in examples]
        vector_mode = _batch_mode(example_sets)
        if nchannels is None:
            nchannels = max([sum(int(cs.num_types) for cs in s) for s in example_sets] or [0])
        dev = torch.device(device) if device is not None else self._device()
        with torch.cuda.device(dev):
            return PackedBatch(example_sets, nchannels, bool(vector_mode), self.radius_scale,
                               bool(self.radius_type_indexed) and check_type_radii,
                               dev, centers=None)

    def _pack_cached(self, example_sets, nchannels, device, check_type_radii=True) -> PackedBatch:
        """``pack`` for the one-shot numpy API, reusing the last batch when the
        same examples come back unchanged (``forward_batch`` followed by
        ``backward_batch`` on the same examples packs once).  A hit needs the
        same set objects AND equal coordinates, radii and types (checked on
        concatenated copies, ~1 ms for C2 vs ~9 ms to pack)."""
        sets = [cs for ss in example_sets for cs in ss]
        key = (tuple(id(cs) for cs in sets), tuple(len(ss) for ss in example_sets),
               tuple(int(cs.num_types) for cs in sets),
               int(nchannels), str(device), float(self.radius_scale),
               bool(self.radius_type_indexed) and check_type_radii)

        def snap():
            cat = (lambda xs: np.concatenate(xs) if xs else np.zeros(0))
            return (cat([np.asarray(cs.coords).reshape(-1) for cs in sets]),
                    cat([np.asarray(cs.radii).reshape(-1) for cs in sets]),
                    cat([np.asarray(cs.type_index).reshape(-1) for cs in sets
                         if getattr(cs, "type_index", None) is not None]),
                    cat([np.asarray(cs.type_vector).reshape(-1) for cs in sets
                         if getattr(cs, "type_vector", None) is not None]),
                    cat([np.asarray(cs.type_radii).reshape(-1) for cs in sets
                         if getattr(cs, "type_radii", None) is not None]))

        # one entry per thread: a batch's workspace (its prepared records) is
        # never shared by calls running concurrently on different threads
        entries = self.__dict__.setdefault("_pack_cache", {})
        tid = threading.get_ident()
        cached = entries.get(tid)
        now = snap()
        if cached is not None and cached[0] == key and len(cached[2]) == len(now) and \
                all(a.shape == b.shape and np.array_equal(a, b) for a, b in zip(cached[2], now)):
            return cached[1]
        pb = self.pack(example_sets, nchannels=nchannels, device=device,
                       check_type_radii=check_type_radii)
        if len(entries) >= 8:  # threads come and go: keep the table small
            entries.clear()
        # the set objects are kept alive with the entry, so their ids stay theirs
        entries[tid] = (key, pb, now, sets)
        return pb

    def __getstate__(self):
        # estimator-style objects pickle / deepcopy as their parameters; the
        # numpy API's pack cache (device buffers) stays behind
        state = dict(self.__dict__)
        state.pop("_pack_cache", None)
        return state

    def _prepare(self, pb: PackedBatch, centers, transforms, npts) -> _native.GmParams:
        if centers is None:
            key = float(self.dimension)
            if getattr(pb, "_origin_key", None) != key:
                pb._default_origins = pb.default_centers - key / 2.0
                pb._origin_key = key
            origins = pb._default_origins
        else:
            origins = np.asarray(centers, np.float64).reshape(-1, 3) - float(self.dimension) / 2.0
        xforms = None
        if transforms is not None:
            if isinstance(transforms, geom.TransformArray):
                xforms = transforms.packed
            elif isinstance(transforms, np.ndarray):
                xforms = transforms.reshape(-1, 15)
            else:
                xforms = np.stack([t.packed() if isinstance(t, geom.Transform)
                                   else np.asarray(t, np.float64).reshape(15)
                                   for t in transforms]) if len(transforms) else np.zeros((0, 15))
        p = self._gm_params(npts)
        pb.set_host_positions(None)
        if xforms is not None and (p.matmul_order_1 < 0 or p.matmul_order_n < 0):
            # numpy's f64 (N,3)@(3,3) rounding could not be reproduced on the
            # device: transform on the host with the
            # reference's own expression (geom.py:105) and ship f64 positions
            _warn_exact_fallback()
            pb.set_host_positions(_host_transformed(pb, xforms))
            xforms = None
        if pb.nexamples <= _native.INLINE_MAX_EXAMPLES:
            # per-call arrays travel inside the prepare launch (no copy)
            pb.ensure_call_buffer(xforms is not None)
            b = pb.gm_batch()
            org = np.ascontiguousarray(origins, np.float64)
            xf = None if xforms is None else np.ascontiguousarray(xforms, np.float64)
            with on_device(pb.device):
                _native.check(_native.lib().gm_prepare_inline(
                    ctypes.byref(p), ctypes.byref(b), pb.workspace.data_ptr(),
                    pb.workspace_bytes, org.ctypes.data, None if xf is None else xf.ctypes.data,
                    stream_handle(pb.device)))
            return p
        pb.set_call_arrays(origins, xforms)
        b = pb.gm_batch()
        with on_device(pb.device):
            _native.check(_native.lib().gm_prepare(
                ctypes.byref(p), ctypes.byref(b), pb.workspace.data_ptr(), pb.workspace_bytes,
                stream_handle(pb.device)))
        return p

    def forward_packed(self, pb: PackedBatch, out=None, centers=None, *,
                       random_translation=0.0, random_rotation=False, rng=None,
                       transforms=None, events=None):
        """Grid a packed batch into a device tensor (N, C, D, D, D).

        Returns ``(out, transforms)``; ``transforms`` is the list of
        ``geom.Transform`` drawn (or given), or None without augmentation.
        """
        self._check_params()
        npts = self.points_per_side()
        shape = (pb.nexamples, pb.nchannels, npts, npts, npts)
        if out is None:
            out = torch.empty(shape, dtype=torch.float32, device=pb.device)
        else:
            _check_device_out(out, shape, pb.device)
        if transforms is None:
            augment = random_rotation or float(random_translation) > 0
            if augment:
                rng = check_rng(rng)
                c = pb.default_centers if centers is None else np.asarray(centers, np.float64)
                transforms = geom.draw_transform_array(c.reshape(-1, 3), float(random_translation),
                                                       bool(random_rotation), rng)
        p = self._prepare(pb, centers, transforms, npts)
        if pb.nexamples and pb.nchannels:
            with on_device(pb.device):
                pb.ensure_fwd_jobs(p)
                if events is not None:
                    events[0].record()
                _native.check(_native.lib().gm_forward(
                    ctypes.byref(p), ctypes.byref(pb._gm), pb.workspace.data_ptr(),
                    out.data_ptr(), stream_handle(pb.device)))
                if events is not None:
                    events[1].record()
        pb._last_params = p
        return out, transforms

    def capture_step(self, pb: PackedBatch, *, augment=True, backward=False, grid_grad=None,
                     out=None):
        """prepare -> forward [-> backward] of ``pb`` captured as CUDA graphs
        (``graph.GraphStep``): each ``run()`` is one input copy + one replay."""
        from .graph import GraphStep
        return GraphStep(self, pb, augment=augment, backward=backward, grid_grad=grid_grad,
                         out=out)

    def backward_packed(self, pb: PackedBatch, grid_grad, centers=None, transforms=None,
                        reuse_prepared=False, coord_grad=None, type_grad=None, events=None):
        """Batched backward over every set of a packed batch.

        ``grid_grad`` is a (N, C, D, D, D) float32 CUDA tensor.  Coordinates
        are taken in the frame of ``transforms`` (the forward's); with
        ``reuse_prepared=True`` the positions of the last ``forward_packed``
        are used as-is.  Returns ``(coord_grad (natoms,3), type_grad
        (nweights,) or None)`` as float32 CUDA tensors in packed atom order.
        """
        self._check_params()
        npts = self.points_per_side()
        shape = (pb.nexamples, pb.nchannels, npts, npts, npts)
        if not self.binary:
            _check_device_in(grid_grad, shape, pb.device, "grid_grad")
        if reuse_prepared and getattr(pb, "_last_params", None) is not None:
            p = pb._last_params
        else:
            p = self._prepare(pb, centers, transforms, npts)
        if coord_grad is None:
            coord_grad = torch.empty((pb.natoms, 3), dtype=torch.float32, device=pb.device)
        if pb.vector_mode and type_grad is None:
            type_grad = torch.empty((pb.nweights,), dtype=torch.float32, device=pb.device)
        with on_device(pb.device):
            if events is not None:
                events[0].record()
            _native.check(_native.lib().gm_backward(
                ctypes.byref(p), ctypes.byref(pb._gm), pb.workspace.data_ptr(),
                None if self.binary else grid_grad.data_ptr(), coord_grad.data_ptr(),
                type_grad.data_ptr() if pb.vector_mode else None, stream_handle(pb.device)))
            if events is not None:
                events[1].record()
        return coord_grad, (type_grad if pb.vector_mode else None)

    # -- forward / backward (voxelizer.py:203-301) --

    def forward(self, atoms, center=None, out=None, *, random_translation=0.0,
                random_rotation=False, rng=None):
        """Voxelize one coordinate set into a (C, D, D, D) float32 grid."""
        if not is_coordinate_set(atoms):
            raise TypeError("atoms must be a CoordinateSet")
        npts = self.points_per_side()
        nch = int(atoms.num_types)
        if center is None:
            center = atoms.centroid()
        shape = (nch, npts, npts, npts)
        arr = self._validate_out(out, shape)
        centers = check_vector3(center, "center").reshape(1, 3)
        return self._run(True, [[atoms]], centers, arr, shape,
                         random_translation, random_rotation, rng)

    def forward_batch(self, examples, out=None, centers=None, *, random_translation=0.0,
                      random_rotation=False, rng=None, return_transforms=False):
        """Voxelize a batch into (N, C, D, D, D); one slab per example."""
        example_sets = [coord_sets_of(ex) for ex in examples]
        if not example_sets:
            raise ValueError("forward_batch needs at least one example")
        npts = self.points_per_side()
        nch = 0
        for sets in example_sets:
            c = sum(int(cs.num_types) for cs in sets)
            if c:
                if nch and c != nch:
                    raise ValueError(f"examples disagree on channel count: {nch} vs {c}")
                nch = c
        if nch == 0:
            if out is None:
                raise ValueError("cannot infer channel count from empty examples; pass out")
            nch = tuple(_unwrap(out).shape)[1]
        n = len(example_sets)
        shape = (n, nch, npts, npts, npts)
        arr = self._validate_out(out, shape)
        if centers is None:
            cen = None
        else:
            cen = np.asarray(centers, dtype=np.float64)
            if cen.shape != (n, 3):
                raise ValueError(f"centers must have shape ({n}, 3), got {cen.shape}")
        res, xf = self._run(False, example_sets, cen, arr, shape, random_translation,
                            random_rotation, rng, want_transforms=True)
        return (res, xf) if return_transforms else res

    def _validate_out(self, out, shape):
        """voxelizer.py:320-333 (numpy / Grid view) plus torch CUDA tensors."""
        if out is None:
            return None
        arr = _unwrap(out)
        if _is_tensor(arr):
            if tuple(arr.shape) != shape:
                raise ValueError(f"out has shape {tuple(arr.shape)}, expected {shape}")
            if arr.dtype != torch.float32:
                raise TypeError(f"out must be float32, got {arr.dtype}")
            if not arr.is_contiguous():
                raise ValueError("out must be C-contiguous")
            return arr
        if not isinstance(arr, np.ndarray):
            raise TypeError("out must be a numpy array or grid")
        if arr.shape != shape:
            raise ValueError(f"out has shape {arr.shape}, expected {shape}")
        if arr.dtype != np.float32:
            raise TypeError(f"out must be float32, got {arr.dtype}")
        if not arr.flags.c_contiguous:
            raise ValueError("out must be C-contiguous")
        return arr

    def _run(self, single, example_sets, centers, arr, shape, random_translation,
             random_rotation, rng, want_transforms=False):
        """voxelizer.py:335-435 on the device.  Returns the output (same object
        as ``arr`` when given) and the transforms drawn."""
        self._check_params()
        augment = random_rotation or float(random_translation) > 0
        if augment:
            rng = check_rng(rng)
        vector_mode = _batch_mode(example_sets)
        if vector_mode is None:
            # nothing but empty sets: a zero grid.  The reference returns
            # before its per-example make_transform loop (voxelizer.py:351-352),
            # so no variate is drawn and the caller's generator is untouched.
            if arr is None:
                arr = np.zeros(shape, dtype=np.float32)
            elif _is_tensor(arr):
                arr.zero_()
            else:
                arr[...] = 0.0
            return (arr, None) if want_transforms else arr
        nch = shape[0] if single else shape[1]
        dev = arr.device if _is_tensor(arr) else self._device()
        pb = self._pack_cached(example_sets, nch, dev)
        dshape = (1,) + shape if single else shape
        if _is_tensor(arr):
            dout = arr.view(dshape)
        else:
            dout = torch.empty(dshape, dtype=torch.float32, device=dev)
        _, xf = self.forward_packed(pb, dout, centers=centers,
                                    random_translation=random_translation,
                                    random_rotation=random_rotation, rng=rng)
        if _is_tensor(arr):
            result = arr
        else:
            # pooled pinned block, or chunked multi-threaded copy-out (hostio.py)
            result = (hostio.grid_to_numpy(dout.view(shape)) if arr is None
                      else hostio.to_host(dout.view(shape), out=arr))
        return (result, xf) if want_transforms else result

    def backward(self, atoms, grid_grad, center=None):
        """Map grid-value gradients back to the atoms of one set.

        Returns ``(coord_grad (N,3), type_grad (N,T) or None)`` float32 --
        numpy arrays, or CUDA tensors when ``grid_grad`` is a CUDA tensor.
        """
        if not is_coordinate_set(atoms):
            raise TypeError("atoms must be a CoordinateSet")
        self._check_params()
        npts = self.points_per_side()
        gg = _unwrap(grid_grad)
        expected = (int(atoms.num_types), npts, npts, npts)
        if tuple(gg.shape) != expected:
            raise ValueError(f"grid_grad shape {tuple(gg.shape)} does not match {expected}")
        if center is None:
            center = atoms.centroid()
        center = check_vector3(center, "center")
        n = int(atoms.coords.shape[0])
        vector = getattr(atoms, "type_vector", None) is not None
        as_tensor = _is_tensor(gg)
        if self.binary or n == 0:
            cg = np.zeros((n, 3), np.float32)
            tg = np.zeros((n, int(atoms.num_types)), np.float32) if vector else None
            if as_tensor:
                cg = torch.from_numpy(cg).to(gg.device)
                tg = torch.from_numpy(tg).to(gg.device) if tg is not None else None
            return cg, tg
        dev = gg.device if as_tensor else self._device()
        pb = self.pack([[atoms]], nchannels=int(atoms.num_types), device=dev)
        if as_tensor:
            dgg = gg.to(torch.float32).contiguous().view((1,) + expected)
        else:
            dgg = hostio.to_device(gg, dev).view((1,) + expected)
        cg, tg = self.backward_packed(pb, dgg, centers=center.reshape(1, 3))
        if vector:
            tg = tg.view(n, int(atoms.num_types))
        if as_tensor:
            return cg, tg
        return cg.cpu().numpy(), (tg.cpu().numpy() if tg is not None else None)

    def backward_batch(self, examples, grid_grad, centers=None, transforms=None,
                       input_frame=False):
        """Backward of ``forward_batch`` over every (example, set).

        ``grid_grad`` (N, C, D, D, D) numpy or CUDA tensor; ``centers`` and
        ``transforms`` as used/returned by ``forward_batch(...,
        return_transforms=True)``.  Returns a list (one per example) of lists
        (one per set) of ``(coord_grad, type_grad)``.  With
        ``input_frame=True`` coordinate gradients are rotated back into the
        input frame (d/dx = R^T d/dx'), i.e. the gradient with respect to the
        untransformed coordinates.
        """
        example_sets = [coord_sets_of(ex) for ex in examples]
        self._check_params()
        npts = self.points_per_side()
        gg = _unwrap(grid_grad)
        nch = tuple(gg.shape)[1]
        expected = (len(example_sets), nch, npts, npts, npts)
        if tuple(gg.shape) != expected:
            raise ValueError(f"grid_grad shape {tuple(gg.shape)} does not match {expected}")
        as_tensor = _is_tensor(gg)
        dev = gg.device if as_tensor else self._device()
        pb = self._pack_cached(example_sets, nch, dev, check_type_radii=not self.binary)
        if as_tensor:
            dgg = gg.to(torch.float32).contiguous()
        else:
            dgg = hostio.to_device(gg, dev)
        cen = None if centers is None else np.asarray(centers, np.float64).reshape(-1, 3)
        cg, tg = self.backward_packed(pb, dgg, centers=cen, transforms=transforms)
        if not as_tensor:
            cg = cg.cpu().numpy()
            tg = tg.cpu().numpy() if tg is not None else None
        out = [[] for _ in example_sets]
        for (e, choff, cs, a0, w0) in pb.placed:
            na, nt = int(cs.coords.shape[0]), int(cs.num_types)
            c = cg[a0:a0 + na]
            if input_frame and transforms is not None:
                # d/dx = R^T d/dx' (row vectors: g R), in f64 then rounded once
                R = _rotation_of(transforms[e])
                c = ((c.double() @ torch.from_numpy(R).to(c.device)).float() if as_tensor
                     else (c.astype(np.float64) @ R).astype(np.float32))
            t = None
            if pb.vector_mode:
                t = tg[w0:w0 + na * nt].reshape(na, nt)
            out[e].append((c, t))
        return out


_FALLBACK_WARNED = [False]


def _warn_exact_fallback() -> None:
    if not _FALLBACK_WARNED[0]:
        import warnings

        warnings.warn("numpy's float64 matmul rounding could not be calibrated on this host; "
                      "augmented coordinates are transformed on the host (exact, slower)",
                      RuntimeWarning, stacklevel=3)
        _FALLBACK_WARNED[0] = True


def _host_transformed(pb: PackedBatch, xforms) -> np.ndarray:
    """(natoms, 3) float64 transformed coordinates, set by set, with the
    reference's expression ((x - c) @ R.T + c) + t (geom.py:105 via
    voxelizer.py:366-368): the same numpy matmul call per set, so the same
    BLAS rounding whatever its FMA order."""
    xf = np.asarray(xforms, np.float64).reshape(-1, 15)
    pos = np.zeros((pb.natoms, 3), np.float64)
    for (e, _choff, cs, a0, _w0) in pb.placed:
        n = int(cs.coords.shape[0])
        if not n:
            continue
        R = np.ascontiguousarray(xf[e, :9]).reshape(3, 3)
        c, t = xf[e, 9:12], xf[e, 12:15]
        pos[a0:a0 + n] = (cs.coords.astype(np.float64) - c) @ R.T + c + t
    return pos


def _rotation_of(t) -> np.ndarray:
    if isinstance(t, geom.Transform):
        return t.rotation.rotation_matrix()
    if hasattr(t, "rotation_matrix"):
        return t.rotation_matrix()
    return np.asarray(t, np.float64).reshape(15)[:9].reshape(3, 3)


def _batch_mode(example_sets):
    """voxelizer.py:342-352: None (all empty), False (index) or True (vector)."""
    mode = None
    for sets in example_sets:
        for cs in sets:
            if cs.coords.shape[0] == 0:
                continue
            vec = getattr(cs, "type_vector", None) is not None
            if mode is None:
                mode = vec
            elif mode != vec:
                raise ValueError("cannot mix index- and vector-typed sets in one batch")
    return mode


def _check_device_out(t, shape, device):
    if not _is_tensor(t) or t.device != device or t.dtype != torch.float32 \
            or not t.is_contiguous() or tuple(t.shape) != shape:
        raise ValueError(f"out must be a contiguous float32 tensor of shape {shape} on {device}")


def _check_device_in(t, shape, device, name):
    if not _is_tensor(t) or t.device != device or t.dtype != torch.float32 \
            or not t.is_contiguous() or tuple(t.shape) != shape:
        raise ValueError(f"{name} must be a contiguous float32 tensor of shape {shape} "
                         f"on {device}")


def save_grid(path, grid, origin=None, resolution=None, channel_labels=None, extra=None) -> str:
    """NPY + JSON sidecar export (voxelizer.py:438-465); accepts CUDA tensors
    (streamed device -> pinned -> file, see export.py)."""
    return export.save_grid(path, grid, origin=origin, resolution=resolution,
                            channel_labels=channel_labels, extra=extra)

"""A whole gridding step captured once as a CUDA graph, replayed per call.

The reference's training loop calls ``GridMaker.forward`` (and ``backward``)
once per batch (/root/reference/pkg/src/voxmol/voxelizer.py:203-301).  For
the large batches of C2 the device time dominates; for small batches (C1: one
ligand, a serving-style call) the step is a few tens of microseconds of
device work behind three C-ABI calls, each with its own argument packing and
launch.  ``GraphStep`` captures prepare -> forward [-> backward] for one
packed batch once and replays it: a call is one host->device copy of the
call's origins and transforms (18 float64 per example, from a fixed pinned
buffer, a node of the graph) plus the recorded launches.  The kernels, their
arguments and their PDL edges are the eager path's, so the outputs are the
eager path's bit for bit (tests/test_gpu_graph.py).

Two graphs alternate over two pinned buffers, so the host fills call k+1's
inputs while call k may still be copying its own.  The outputs
(``out``, ``coord_grad``, ``type_grad``) are static tensors that every replay
rewrites: consume (or copy) them before the next ``run`` on another stream.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native, geom
from .packing import PackedBatch, stream_handle
from .validation import check_rng


class GraphStep:
    """prepare -> forward [-> backward] of ``pb`` as replayable CUDA graphs.

    ``augment``: the step applies a per-example transform each call (random
    draws in ``run``, or given ``transforms``); without it the grids are taken
    at the centers, as ``forward_packed`` without transforms.
    ``backward``: also run the backward of ``grid_grad`` (a static (N,C,D,D,D)
    float32 tensor the caller fills in place, or passes to ``run``).
    """

    def __init__(self, gm, pb: PackedBatch, *, augment: bool = True, backward: bool = False,
                 grid_grad: torch.Tensor | None = None, out: torch.Tensor | None = None):
        if pb.device.type != "cuda":
            raise ValueError("GraphStep needs a CUDA packed batch")
        gm._check_params()
        self.gm, self.pb = gm, pb
        self.augment = bool(augment)
        self.backward = bool(backward)
        npts = gm.points_per_side()
        n = pb.nexamples
        self.shape = (n, pb.nchannels, npts, npts, npts)
        dev = pb.device
        self.out = out if out is not None else torch.empty(self.shape, dtype=torch.float32,
                                                           device=dev)
        if tuple(self.out.shape) != self.shape or self.out.dtype != torch.float32 \
                or not self.out.is_contiguous() or self.out.device != dev:
            raise ValueError(f"out must be a contiguous float32 {self.shape} tensor on {dev}")
        self.grid_grad = None
        self.coord_grad = self.type_grad = None
        if self.backward:
            if not gm.binary:
                if grid_grad is None:
                    grid_grad = torch.zeros(self.shape, dtype=torch.float32, device=dev)
                if tuple(grid_grad.shape) != self.shape or grid_grad.dtype != torch.float32 \
                        or not grid_grad.is_contiguous() or grid_grad.device != dev:
                    raise ValueError(f"grid_grad must be a contiguous float32 {self.shape} "
                                     f"tensor on {dev}")
                self.grid_grad = grid_grad
            self.coord_grad = torch.empty((pb.natoms, 3), dtype=torch.float32, device=dev)
            if pb.vector_mode:
                self.type_grad = torch.empty((pb.nweights,), dtype=torch.float32, device=dev)
        self._m = (18 if self.augment else 3) * n
        self._host = [torch.zeros(max(self._m, 1), dtype=torch.float64, pin_memory=True)
                      for _ in range(2)]
        self._done = [None, None]
        self._k = 0
        self._params = gm._gm_params(npts)
        if self.augment and (self._params.matmul_order_1 < 0 or self._params.matmul_order_n < 0):
            import warnings

            # the captured prepare pass transforms on the device; the eager path
            # falls back to host-transformed positions instead (voxelizer._prepare)
            warnings.warn("numpy's float64 matmul rounding could not be calibrated on this "
                          "host: the graph-captured transform may differ from numpy's in the "
                          "last bit (binary occupancy is then not guaranteed bit-exact)",
                          RuntimeWarning, stacklevel=2)
        pb.ensure_call_buffer(self.augment)
        self._batch = pb.gm_batch()
        self._origin_shift = float(gm.dimension) / 2.0
        # warm-up outside capture: job table upload, kernel attributes, and
        # identity inputs so the captured launches read defined memory
        for h in self._host:
            self._fill(h.numpy(), None, None)
        with torch.cuda.device(dev):
            pb.ensure_fwd_jobs(self._params)
            self._record(self._host[0])
            torch.cuda.synchronize(dev)
            self._graphs = []
            for h in self._host:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    self._record(h)
                self._graphs.append(g)
            torch.cuda.synchronize(dev)

    # -- capture --------------------------------------------------------------
    def _record(self, host: torch.Tensor) -> None:
        pb, p, b = self.pb, self._params, self._batch
        lib = _native.lib()
        if self._m:
            pb._percall[:self._m].copy_(host[:self._m], non_blocking=True)
        s = stream_handle(pb.device)
        ws = pb.workspace.data_ptr()
        _native.check(lib.gm_prepare(ctypes.byref(p), ctypes.byref(b), ws, pb.workspace_bytes, s))
        if pb.nexamples and pb.nchannels:
            _native.check(lib.gm_forward(ctypes.byref(p), ctypes.byref(b), ws,
                                         self.out.data_ptr(), s))
        if self.backward:
            _native.check(lib.gm_backward(
                ctypes.byref(p), ctypes.byref(b), ws,
                None if self.grid_grad is None else self.grid_grad.data_ptr(),
                self.coord_grad.data_ptr(),
                None if self.type_grad is None else self.type_grad.data_ptr(), s))

    def _fill(self, h: np.ndarray, centers, xforms) -> None:
        n = self.pb.nexamples
        c = self.pb.default_centers if centers is None else \
            np.asarray(centers, np.float64).reshape(n, 3)
        h[:3 * n] = (c - self._origin_shift).reshape(-1)
        if self.augment:
            if xforms is None:  # identity rotation about the center, no shift
                x = np.zeros((n, 15))
                x[:, [0, 4, 8]] = 1.0
                x[:, 9:12] = c
                xforms = x
            h[3 * n:18 * n] = np.asarray(xforms, np.float64).reshape(-1)

    # -- per call -------------------------------------------------------------
    def run(self, *, transforms=None, centers=None, random_rotation=False,
            random_translation=0.0, rng=None, grid_grad=None):
        """One step.  Returns ``(out, transforms)`` (forward only) or
        ``(out, coord_grad, type_grad, transforms)``; the tensors are this
        step's static outputs."""
        n = self.pb.nexamples
        xforms = None
        if self.augment:
            if transforms is None and (random_rotation or float(random_translation) > 0):
                rng = check_rng(rng)
                c = self.pb.default_centers if centers is None else np.asarray(centers, np.float64)
                transforms = geom.draw_transform_array(c.reshape(-1, 3), float(random_translation),
                                                       bool(random_rotation), rng)
            if transforms is not None:
                xforms = (transforms.packed if isinstance(transforms, geom.TransformArray)
                          else np.stack([t.packed() if isinstance(t, geom.Transform)
                                         else np.asarray(t, np.float64).reshape(15)
                                         for t in transforms]))
                if xforms.shape != (n, 15):
                    raise ValueError(f"need {n} transforms, got {xforms.shape[0]}")
        elif transforms is not None or random_rotation or float(random_translation) > 0:
            raise ValueError("this GraphStep was captured without augment")
        k = self._k
        self._k ^= 1
        if self._done[k] is not None:
            self._done[k].synchronize()  # the replay that last read this buffer
        self._fill(self._host[k].numpy(), centers, xforms)
        dev = self.pb.device
        if grid_grad is not None:
            if self.grid_grad is None:
                raise ValueError("this GraphStep has no backward over grid_grad")
            if grid_grad.data_ptr() != self.grid_grad.data_ptr():
                self.grid_grad.copy_(grid_grad)
        self._graphs[k].replay()
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(dev))
        self._done[k] = ev
        self.pb._last_params = self._params
        if self.backward:
            return self.out, self.coord_grad, self.type_grad, transforms
        return self.out, transforms

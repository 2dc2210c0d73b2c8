"""Drop-in for the reference's kernel module ``voxmol._kernels``.

Same four functions, same argument names, order, dtypes and return values as
/root/reference/pkg/src/voxmol/_kernels.py (forward_index_sets 33-36,
forward_vector_sets 116-120, backward_index 209-210, backward_vector
258-260), operating on host numpy arrays exactly like the numba kernels.
Each call goes through the C ABI's ``*_host`` entry points
(include/gridmaker_b200.h), which stage the arrays to the GPU, run the
sm_100a kernels and copy the results back.  INTEGRATION.md shows the
one-line switch in voxmol/voxelizer.py.

Differences by design: ``out`` need not be pre-zeroed (every voxel is
written), and the kernels release the GIL for the duration of the call.
"""

from __future__ import annotations

import numpy as np

from . import _native


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _p(a):
    return a.ctypes.data if a is not None and a.size else None


def forward_index_sets(out, coords, radii, tidx, set_start, set_end, set_example, set_choff,
                       set_t, origins, res, grm, rmult, binary):
    """_kernels.py:33-113 on the GPU; writes ``out`` (N, C, D, D, D) float32."""
    if out.dtype != np.float32 or not out.flags.c_contiguous:
        raise TypeError("out must be a C-contiguous float32 array")
    coords, radii = _c(coords, np.float64), _c(radii, np.float64)
    tidx = _c(tidx, np.int64)
    sets = [_c(a, np.int64) for a in (set_start, set_end, set_example, set_choff, set_t)]
    origins = _c(origins, np.float64)
    n, nch, d = out.shape[0], out.shape[1], out.shape[2]
    _native.check(_native.lib().gm_forward_index_sets_host(
        out.ctypes.data, n, nch, d, _p(coords), _p(radii), _p(tidx), coords.shape[0],
        _p(sets[0]), _p(sets[1]), _p(sets[2]), _p(sets[3]), _p(sets[4]), sets[0].shape[0],
        origins.ctypes.data, float(res), float(grm), float(rmult), int(bool(binary))))


def forward_vector_sets(out, coords, weights_flat, w_start, atom_radii, type_radii_flat, tr_start,
                        radius_type_indexed, set_start, set_end, set_example, set_choff, set_t,
                        origins, res, grm, rmult, binary):
    """_kernels.py:116-206 on the GPU; writes ``out`` (N, C, D, D, D) float32."""
    if out.dtype != np.float32 or not out.flags.c_contiguous:
        raise TypeError("out must be a C-contiguous float32 array")
    coords = _c(coords, np.float64)
    weights_flat, atom_radii = _c(weights_flat, np.float64), _c(atom_radii, np.float64)
    type_radii_flat = _c(type_radii_flat, np.float64)
    w_start, tr_start = _c(w_start, np.int64), _c(tr_start, np.int64)
    sets = [_c(a, np.int64) for a in (set_start, set_end, set_example, set_choff, set_t)]
    origins = _c(origins, np.float64)
    n, nch, d = out.shape[0], out.shape[1], out.shape[2]
    _native.check(_native.lib().gm_forward_vector_sets_host(
        out.ctypes.data, n, nch, d, _p(coords), coords.shape[0], _p(weights_flat),
        weights_flat.shape[0], _p(w_start), _p(atom_radii), _p(type_radii_flat),
        type_radii_flat.shape[0], _p(tr_start), int(bool(radius_type_indexed)),
        _p(sets[0]), _p(sets[1]), _p(sets[2]), _p(sets[3]), _p(sets[4]), sets[0].shape[0],
        origins.ctypes.data, float(res), float(grm), float(rmult), int(bool(binary))))


def backward_index(coords, radii, tidx, grid_grad, origin, res, grm, rmult):
    """_kernels.py:209-255 on the GPU -> coord_grad (n, 3) float64."""
    coords, radii, tidx = _c(coords, np.float64), _c(radii, np.float64), _c(tidx, np.int64)
    gg = _c(grid_grad, np.float32)
    origin = _c(origin, np.float64)
    n = coords.shape[0]
    cg = np.zeros((n, 3), np.float64)
    _native.check(_native.lib().gm_backward_index_host(
        cg.ctypes.data, _p(coords), _p(radii), _p(tidx), n, gg.ctypes.data, gg.shape[0],
        gg.shape[1], origin.ctypes.data, float(res), float(grm), float(rmult)))
    return cg


def backward_vector(coords, atom_radii, weights, grid_grad, type_radii, radius_type_indexed,
                    origin, res, grm, rmult):
    """_kernels.py:258-314 on the GPU -> (coord_grad (n, 3), type_grad (n, T)) float64."""
    coords, atom_radii = _c(coords, np.float64), _c(atom_radii, np.float64)
    weights = _c(weights, np.float64)
    gg = _c(grid_grad, np.float32)
    type_radii = _c(type_radii, np.float64)
    origin = _c(origin, np.float64)
    n, nt = weights.shape[0], weights.shape[1]
    cg = np.zeros((n, 3), np.float64)
    tg = np.zeros((n, nt), np.float64)
    _native.check(_native.lib().gm_backward_vector_host(
        cg.ctypes.data, tg.ctypes.data, _p(coords), _p(atom_radii), _p(weights), n, nt,
        gg.ctypes.data, gg.shape[1], _p(type_radii), int(bool(radius_type_indexed)),
        origin.ctypes.data, float(res), float(grm), float(rmult)))
    return cg, tg

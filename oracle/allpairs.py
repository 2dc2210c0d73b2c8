"""All-pairs float64 oracle -- TEST INFRASTRUCTURE ONLY.

An independent second checker that follows the density *definitions* used
by the reference's own numpy oracle (``/root/reference/pkg/tests/oracles.py``:
density 19-29, voxel centres 32-38, all-pairs forward 41-76, seam masking
79-99, finite differences 102-145).  It evaluates every (voxel, atom) pair
over the whole grid, so it exercises the box culling of both the C oracle
and the CUDA path, which it never calls.
"""

from __future__ import annotations

import math

import numpy as np


def npts_for(resolution: float, dimension: float) -> int:
    """Points per axis: round-half-up(dimension / resolution) + 1."""
    return int(math.floor(dimension / resolution + 0.5)) + 1


def shell_radii(r: float, grm: float):
    """(gaussian handoff d0, cutoff dz, quadratic coefficient) for radius r."""
    d0 = grm * r
    dz = r * (1.0 + 2.0 * grm * grm) / (2.0 * grm)
    coef = math.exp(-2.0 * grm * grm) / (d0 - dz) ** 2
    return d0, dz, coef


def density_of_distance(dist, r, grm=1.0, binary=False):
    dist = np.asarray(dist, dtype=np.float64)
    if binary:
        return (dist <= r).astype(np.float64)
    d0, dz, coef = shell_radii(r, grm)
    value = np.zeros_like(dist)
    core = dist <= d0
    tail = (~core) & (dist < dz)
    value[core] = np.exp(-2.0 * dist[core] ** 2 / (r * r))
    value[tail] = coef * (dist[tail] - dz) ** 2
    return value


def voxel_positions(center, resolution, dimension):
    """Axis coordinate vectors (x, y, z) of the voxel centres."""
    n = npts_for(resolution, dimension)
    lo = np.asarray(center, dtype=np.float64).reshape(3) - dimension / 2.0
    steps = resolution * np.arange(n)
    return lo[0] + steps, lo[1] + steps, lo[2] + steps


def _distance_field(axes, p):
    ax, ay, az = axes
    return np.sqrt((ax - p[0])[:, None, None] ** 2 + (ay - p[1])[None, :, None] ** 2
                   + (az - p[2])[None, None, :] ** 2)


def grid_all_pairs(coords, radii, type_index, num_types, center, resolution=0.5,
                   dimension=23.5, grm=1.0, binary=False, radius_scale=1.0,
                   type_vector=None, type_radii=None):
    """(T, D, D, D) float64 grid summed (or max-ed, binary) over every atom."""
    axes = voxel_positions(center, resolution, dimension)
    n = axes[0].shape[0]
    out = np.zeros((num_types, n, n, n))
    pts = np.asarray(coords, dtype=np.float64).reshape(-1, 3)
    rad = np.asarray(radii, dtype=np.float64).reshape(-1) * radius_scale
    combine = np.maximum if binary else np.add
    for a in range(pts.shape[0]):
        dist = _distance_field(axes, pts[a])
        if type_vector is None:
            c = int(type_index[a])
            out[c] = combine(out[c], density_of_distance(dist, rad[a], grm, binary))
            continue
        for c in range(num_types):
            w = float(type_vector[a][c])
            if w == 0.0:
                continue
            r = rad[a] if type_radii is None else radius_scale * float(type_radii[c])
            out[c] = combine(out[c], w * density_of_distance(dist, r, grm, binary))
    return out


def mask_seams(grid_grad, coords, radii, center, resolution=0.5, dimension=23.5,
               grm=1.0, radius_scale=1.0, margin=0.05):
    """Zero gradient voxels within ``margin`` of any atom centre, handoff or cutoff
    shell (the density is only C1 there, so finite differences are O(h))."""
    gg = np.array(grid_grad, dtype=np.float64, copy=True)
    axes = voxel_positions(center, resolution, dimension)
    pts = np.asarray(coords, dtype=np.float64).reshape(-1, 3)
    for a in range(pts.shape[0]):
        r = float(radii[a]) * radius_scale
        d0, dz, _ = shell_radii(r, grm)
        dist = _distance_field(axes, pts[a])
        near = (dist < margin) | (np.abs(dist - d0) < margin) | (np.abs(dist - dz) < margin)
        gg[:, near] = 0.0
    return gg


def central_differences(loss, x, h):
    """d loss / d x by central differences, elementwise over an array."""
    x = np.asarray(x, dtype=np.float64)
    g = np.zeros_like(x)
    for idx in np.ndindex(*x.shape):
        xp = x.copy()
        xm = x.copy()
        xp[idx] += h
        xm[idx] -= h
        g[idx] = (loss(xp) - loss(xm)) / (2.0 * h)
    return g


def relative_errors(analytic, numeric, scale_floor=0.1):
    """|a-n| / max(|a|, |n|, scale_floor * max|n|) (floor >= 1e-8)."""
    a = np.asarray(analytic, dtype=np.float64)
    n = np.asarray(numeric, dtype=np.float64)
    floor = max(scale_floor * float(np.abs(n).max(initial=0.0)), 1e-8)
    return np.abs(a - n) / np.maximum(np.maximum(np.abs(a), np.abs(n)), floor)

"""CPU oracle for the GridMaker hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package, and
only as the checker / CPU baseline.  The product package
(``paper_1912_04822_b200``) never imports it and has no CPU fallback.

Contents
--------
* ``liboracle.so`` (built from ``oracle.c``): a C restatement of the
  reference's numba kernels ``/root/reference/pkg/src/voxmol/_kernels.py``
  (forward_index_sets 33-113, forward_vector_sets 116-206, backward_index
  209-255, backward_vector 258-314) with the same IEEE operation order.
* ``GridOracle``: a restatement of the reference host layer that packs
  CSR arrays and draws transforms (``voxelizer.py:203-301,335-435``,
  ``geom.py:50-136``), then calls the C kernels.
* ``allpairs``: a restatement of the reference's independent numpy oracle
  (``/root/reference/pkg/tests/oracles.py``).

Parity pinning: ``tests/golden/make_golden.py`` ran the live reference
(``voxmol`` from ``/root/reference/pkg/src``) in the build container and
stored its outputs under ``tests/golden/``; ``tests/test_oracle_golden.py``
checks this oracle against them.
"""

from __future__ import annotations

import ctypes
import math
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB = None

_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i64 = ctypes.c_int64
_dbl = ctypes.c_double
_int = ctypes.c_int


def build(force: bool = False) -> Path:
    """Compile liboracle.so with the committed Makefile."""
    so = _HERE / "liboracle.so"
    if force or not so.exists() or so.stat().st_mtime < (_HERE / "oracle.c").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return so


def lib():
    global _LIB
    if _LIB is None:
        so = _HERE / "liboracle.so"
        if not so.exists():
            build()
        L = ctypes.CDLL(str(so))
        L.oracle_forward_index_sets.argtypes = [
            _f32p, _i64, _i64, _f64p, _f64p, _i64p, _i64p, _i64p, _i64p, _i64p, _i64p,
            _i64, _f64p, _dbl, _dbl, _dbl, _int]
        L.oracle_forward_index_sets.restype = None
        L.oracle_forward_vector_sets.argtypes = [
            _f32p, _i64, _i64, _f64p, _f64p, _i64p, _f64p, _f64p, _i64p, _int,
            _i64p, _i64p, _i64p, _i64p, _i64p, _i64, _f64p, _dbl, _dbl, _dbl, _int]
        L.oracle_forward_vector_sets.restype = None
        L.oracle_backward_index.argtypes = [
            _f64p, _f64p, _f64p, _i64p, _i64, _f32p, _i64, _f64p, _dbl, _dbl, _dbl]
        L.oracle_backward_index.restype = None
        L.oracle_backward_vector.argtypes = [
            _f64p, _f64p, _f64p, _f64p, _f64p, _i64, _i64, _f32p, _i64, _f64p, _int,
            _f64p, _dbl, _dbl, _dbl]
        L.oracle_backward_vector.restype = None
        L.oracle_num_threads.restype = _int
        L.oracle_set_num_threads.argtypes = [_int]
        _LIB = L
    return _LIB


def set_num_threads(n: int) -> None:
    lib().oracle_set_num_threads(int(n))


def num_threads() -> int:
    return int(lib().oracle_num_threads())


# ---------------------------------------------------------------- geometry
# Restatement of /root/reference/pkg/src/voxmol/geom.py (host numpy/libm).

def quaternion_rotation_matrix(w, x, y, z) -> np.ndarray:
    """geom.py:50-57 (column-vector convention, float64)."""
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
        [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
        [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)],
    ], dtype=np.float64)


def _normalized(w, x, y, z):
    """geom.py:28-36: renormalise only when |n-1| > 1e-6."""
    n = math.sqrt(w ** 2 + x ** 2 + y ** 2 + z ** 2)
    if abs(n - 1.0) > 1e-6:
        return w / n, x / n, y / n, z / n
    return w, x, y, z


def random_unit_quaternion(rng):
    """geom.py:66-76 (Shoemake)."""
    u1, u2, u3 = rng.random(3)
    a, b = math.sqrt(1.0 - u1), math.sqrt(u1)
    t2, t3 = 2.0 * math.pi * u2, 2.0 * math.pi * u3
    return _normalized(b * math.cos(t3), a * math.sin(t2), a * math.cos(t2), b * math.sin(t3))


def make_transform(center, random_translate, random_rotation, rng):
    """geom.py:121-136 -> (R 3x3, center (3,), translation (3,))."""
    center = np.asarray(center, dtype=np.float64).reshape(3)
    q = random_unit_quaternion(rng) if random_rotation else (1.0, 0.0, 0.0, 0.0)
    if random_translate > 0:
        t = rng.uniform(-random_translate, random_translate, size=3)
    else:
        t = np.zeros(3)
    return quaternion_rotation_matrix(*q), center, np.asarray(t, dtype=np.float64)


def apply_transform(R, center, t, coords64):
    """geom.py:105: ((x - c) @ R.T + c) + t in float64 via numpy."""
    return (coords64 - center) @ R.T + center + t


# ---------------------------------------------------------------- host layer
# Restatement of voxelizer.GridMaker's parameter helpers and _run_batch.

def points_per_side(resolution, dimension) -> int:
    """voxelizer.py:143-146."""
    return int(math.floor(float(dimension) / float(resolution) + 0.5)) + 1


def radius_multiple(grm) -> float:
    """voxelizer.py:148-152."""
    grm = float(grm)
    return (1.0 + 2.0 * grm * grm) / (2.0 * grm)


def _sets_of(example):
    sets = getattr(example, "coord_sets", None)
    if sets is None:
        return [example]
    return list(sets)


def centroid(cs) -> np.ndarray:
    """atomtypes.py:80-84."""
    if cs.coords.shape[0] == 0:
        return np.zeros(3, dtype=np.float64)
    return cs.coords.astype(np.float64).mean(axis=0)


def default_center(sets) -> np.ndarray:
    """voxelizer.py:305-309: centroid of the last non-empty set."""
    for cs in reversed(sets):
        if cs.coords.shape[0]:
            return centroid(cs)
    return np.zeros(3, dtype=np.float64)


class GridOracle:
    """CPU GridMaker with the reference's semantics (forward_batch/backward)."""

    def __init__(self, resolution=0.5, dimension=23.5, binary=False,
                 radius_type_indexed=False, radius_scale=1.0,
                 gaussian_radius_multiple=1.0):
        self.resolution = float(resolution)
        self.dimension = float(dimension)
        self.binary = bool(binary)
        self.radius_type_indexed = bool(radius_type_indexed)
        self.radius_scale = float(radius_scale)
        self.grm = float(gaussian_radius_multiple)

    @property
    def npts(self):
        return points_per_side(self.resolution, self.dimension)

    @property
    def rmult(self):
        return radius_multiple(self.grm)

    def origin(self, center):
        return np.asarray(center, dtype=np.float64).reshape(3) - self.dimension / 2.0

    def place(self, examples, centers=None, random_translation=0.0,
              random_rotation=False, rng=None):
        """voxelizer.py:223-258 + 354-370: centers, origins, transformed f64 coords.

        Returns (example_sets, centers (N,3), origins (N,3), placed) where
        placed is a list of (e, choff, cs, coords64).
        """
        example_sets = [_sets_of(ex) for ex in examples]
        n = len(example_sets)
        if centers is None:
            centers = np.stack([default_center(s) for s in example_sets]) if n else np.zeros((0, 3))
        centers = np.asarray(centers, dtype=np.float64).reshape(n, 3)
        augment = random_rotation or float(random_translation) > 0
        if augment and not isinstance(rng, np.random.Generator):
            rng = np.random.default_rng(rng)
        origins = np.empty((n, 3), dtype=np.float64)
        placed = []
        xforms = []
        for e, sets in enumerate(example_sets):
            origins[e] = self.origin(centers[e])
            xf = make_transform(centers[e], float(random_translation), random_rotation, rng) \
                if augment else None
            xforms.append(xf)
            choff = 0
            for cs in sets:
                c64 = cs.coords.astype(np.float64)
                if xf is not None and cs.coords.shape[0]:
                    c64 = apply_transform(*xf, c64)
                placed.append((e, choff, cs, c64))
                choff += cs.num_types
        return example_sets, centers, origins, placed, xforms

    def forward_batch(self, examples, centers=None, random_translation=0.0,
                      random_rotation=False, rng=None, nch=None):
        example_sets, centers, origins, placed, _ = self.place(
            examples, centers, random_translation, random_rotation, rng)
        if nch is None:
            nch = max(sum(cs.num_types for cs in sets) for sets in example_sets)
        D = self.npts
        out = np.zeros((len(example_sets), nch, D, D, D), dtype=np.float32)
        self.forward_placed(out, placed, origins)
        return out

    def pack_placed(self, placed):
        """voxelizer.py:372-435: the packed CSR arrays of the reference's
        _kernels calls, as a dict (keys = _kernels argument names)."""
        nonempty = [p for p in placed if p[2].coords.shape[0]]
        vector_mode = bool(nonempty) and nonempty[0][2].type_vector is not None
        nsets = len(placed)
        natoms = sum(p[2].coords.shape[0] for p in placed)
        d = dict(coords=np.zeros((natoms, 3), dtype=np.float64),
                 set_start=np.zeros(nsets, np.int64), set_end=np.zeros(nsets, np.int64),
                 set_example=np.zeros(nsets, np.int64), set_choff=np.zeros(nsets, np.int64),
                 set_t=np.zeros(nsets, np.int64), vector_mode=vector_mode)
        pos = 0
        for s, (e, choff, cs, c64) in enumerate(placed):
            na = cs.coords.shape[0]
            d["set_start"][s], d["set_end"][s] = pos, pos + na
            d["set_example"][s], d["set_choff"][s], d["set_t"][s] = e, choff, cs.num_types
            d["coords"][pos:pos + na] = c64
            pos += na
        scale = self.radius_scale
        if vector_mode:
            wtot = sum(p[2].coords.shape[0] * p[2].num_types for p in placed)
            d["weights_flat"] = np.zeros(wtot, np.float64)
            d["w_start"] = np.zeros(nsets, np.int64)
            d["type_radii_flat"] = np.zeros(max(1, sum(p[2].num_types for p in placed)),
                                            np.float64)
            d["tr_start"] = np.zeros(nsets, np.int64)
            d["atom_radii"] = np.zeros(natoms, np.float64)
            wpos = tpos = 0
            for s, (e, choff, cs, c64) in enumerate(placed):
                na, nt = cs.coords.shape[0], cs.num_types
                d["w_start"][s] = wpos
                if na:
                    d["weights_flat"][wpos:wpos + na * nt] = \
                        cs.type_vector.astype(np.float64).ravel()
                wpos += na * nt
                d["tr_start"][s] = tpos
                if na and self.radius_type_indexed:
                    d["type_radii_flat"][tpos:tpos + nt] = cs.type_radii.astype(np.float64) * scale
                else:
                    d["type_radii_flat"][tpos:tpos + nt] = 1.0
                tpos += nt
                d["atom_radii"][d["set_start"][s]:d["set_end"][s]] = \
                    cs.radii.astype(np.float64) * scale
        else:
            d["radii"] = np.zeros(natoms, np.float64)
            d["tidx"] = np.zeros(natoms, np.int64)
            for s, (e, choff, cs, c64) in enumerate(placed):
                if cs.coords.shape[0] == 0:
                    continue
                d["radii"][d["set_start"][s]:d["set_end"][s]] = cs.radii.astype(np.float64) * scale
                d["tidx"][d["set_start"][s]:d["set_end"][s]] = cs.type_index
        return d

    def forward_placed(self, out, placed, origins):
        """voxelizer.py:372-435: pack CSR arrays and dispatch to the C kernels."""
        if not any(p[2].coords.shape[0] for p in placed):
            return out
        d = self.pack_placed(placed)
        L = lib()
        origins = np.ascontiguousarray(origins, dtype=np.float64)
        D = out.shape[2]
        sets = (d["set_start"], d["set_end"], d["set_example"], d["set_choff"], d["set_t"])
        if d["vector_mode"]:
            L.oracle_forward_vector_sets(
                out, out.shape[1], D, d["coords"], d["weights_flat"], d["w_start"],
                d["atom_radii"], d["type_radii_flat"], d["tr_start"],
                int(self.radius_type_indexed), *sets, len(placed), origins, self.resolution,
                self.grm, self.rmult, int(self.binary))
        else:
            L.oracle_forward_index_sets(
                out, out.shape[1], D, d["coords"], d["radii"], d["tidx"], *sets, len(placed),
                origins, self.resolution, self.grm, self.rmult, int(self.binary))
        return out

    def forward(self, cs, center=None, random_translation=0.0, random_rotation=False, rng=None):
        """voxelizer.py:203-221 (default center = the set's own centroid)."""
        if center is None:
            center = centroid(cs)
        out = self.forward_batch([cs], centers=np.asarray(center, np.float64).reshape(1, 3),
                                 random_translation=random_translation,
                                 random_rotation=random_rotation, rng=rng, nch=cs.num_types)
        return out[0]

    def backward(self, cs, grid_grad, center=None, coords64=None):
        """voxelizer.py:260-301.  ``coords64`` overrides the set's coordinates
        (the transformed frame a batched forward used)."""
        if center is None:
            center = centroid(cs)
        origin = np.ascontiguousarray(self.origin(center))
        n = cs.coords.shape[0]
        coords = np.ascontiguousarray(cs.coords.astype(np.float64) if coords64 is None
                                      else coords64, dtype=np.float64)
        radii = np.ascontiguousarray(cs.radii.astype(np.float64) * self.radius_scale)
        gg = np.ascontiguousarray(grid_grad, dtype=np.float32)
        D = self.npts
        vector = cs.type_vector is not None
        if self.binary:
            cg = np.zeros((n, 3), np.float32)
            return cg, (np.zeros((n, cs.num_types), np.float32) if vector else None)
        cg = np.zeros((n, 3), np.float64)
        L = lib()
        if vector:
            nt = cs.num_types
            tg = np.zeros((n, nt), np.float64)
            if self.radius_type_indexed:
                tr = cs.type_radii.astype(np.float64) * self.radius_scale
            else:
                tr = np.ones(nt, np.float64)
            L.oracle_backward_vector(
                cg, tg, coords, radii, np.ascontiguousarray(cs.type_vector, dtype=np.float64),
                n, nt, gg, D, np.ascontiguousarray(tr), int(self.radius_type_indexed),
                origin, self.resolution, self.grm, self.rmult)
            return cg.astype(np.float32), tg.astype(np.float32)
        L.oracle_backward_index(cg, coords, radii, np.ascontiguousarray(cs.type_index, np.int64),
                                n, gg, D, origin, self.resolution, self.grm, self.rmult)
        return cg.astype(np.float32), None

    def backward_batch(self, examples, grid_grad, centers=None, random_translation=0.0,
                       random_rotation=False, rng=None):
        """Per-(example, set) loop of backward() in the forward's frame: the
        reference has no batch backward; this is the loop its
        users write, with the forward's centers and transformed coordinates."""
        example_sets, centers, origins, placed, _ = self.place(
            examples, centers, random_translation, random_rotation, rng)
        cgs, tgs = [], []
        for (e, choff, cs, c64) in placed:
            nt = cs.num_types
            cg, tg = self.backward(cs, grid_grad[e, choff:choff + nt], center=centers[e],
                                   coords64=c64)
            cgs.append(cg)
            tgs.append(tg)
        return cgs, tgs

"""Rigid transforms for augmentation: quaternion rotation about a centre plus
translation.

Host-side API mirror of /root/reference/pkg/src/voxmol/geom.py
(Quaternion 19-60, random_unit_quaternion 66-76, Transform 83-118,
make_transform 121-136, transform_example 139-151).  The random draws and
the rotation matrix are computed on the host with the reference's formulas
so that a seeded stream yields bit-identical transforms; the per-atom
application inside ``GridMaker.forward_batch`` runs on the GPU
(``k_prepare_static`` in csrc/prepare.cu) in the FMA order numpy's matmul uses
on this host (see ``matmul_order``).
"""

from __future__ import annotations

import ctypes
import ctypes.util
import math
from dataclasses import dataclass, field

import numpy as np

from .validation import check_non_negative, check_rng, check_vector3


@dataclass(frozen=True)
class Quaternion:
    """Unit quaternion (w, x, y, z); renormalised when |norm - 1| > 1e-6."""

    w: float = 1.0
    x: float = 0.0
    y: float = 0.0
    z: float = 0.0

    def __post_init__(self):
        n = self.norm
        if n == 0.0 or not math.isfinite(n):
            raise ValueError("cannot normalize a zero or non-finite quaternion")
        if abs(n - 1.0) > 1e-6:
            for name in ("w", "x", "y", "z"):
                object.__setattr__(self, name, getattr(self, name) / n)

    @property
    def norm(self) -> float:
        return math.sqrt(self.w ** 2 + self.x ** 2 + self.y ** 2 + self.z ** 2)

    def conjugate(self) -> "Quaternion":
        return Quaternion(self.w, -self.x, -self.y, -self.z)

    @property
    def angle(self) -> float:
        """Rotation angle in [0, pi]."""
        return 2.0 * math.acos(min(1.0, abs(self.w)))

    def rotation_matrix(self) -> np.ndarray:
        """3x3 float64 matrix acting on column vectors."""
        return np.array(_rotation_rows(self.w, self.x, self.y, self.z), dtype=np.float64)

    def rotate(self, vec) -> np.ndarray:
        return self.rotation_matrix() @ np.asarray(vec, dtype=np.float64)


def _rotation_rows(w, x, y, z):
    # Same Python-float expressions as geom.py:53-57, so R is bit-identical.
    return [
        [1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
        [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
        [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)],
    ]


IDENTITY_QUATERNION = Quaternion(1.0, 0.0, 0.0, 0.0)


def _quaternion_from_uniforms(u1, u2, u3) -> Quaternion:
    a, b = math.sqrt(1.0 - u1), math.sqrt(u1)
    t2, t3 = 2.0 * math.pi * u2, 2.0 * math.pi * u3
    return Quaternion(b * math.cos(t3), a * math.sin(t2), a * math.cos(t2), b * math.sin(t3))


def random_unit_quaternion(rng=None) -> Quaternion:
    """Uniform over SO(3) from three uniform variates (Shoemake)."""
    u1, u2, u3 = check_rng(rng).random(3)
    return _quaternion_from_uniforms(u1, u2, u3)


@dataclass(frozen=True)
class Transform:
    """x -> R (x - center) + center + translation."""

    rotation: Quaternion = field(default_factory=Quaternion)
    center: np.ndarray = None
    translation: np.ndarray = None

    def __post_init__(self):
        for name in ("center", "translation"):
            v = getattr(self, name)
            object.__setattr__(self, name, check_vector3((0.0, 0.0, 0.0) if v is None else v))

    def forward(self, coords_in, coords_out=None) -> np.ndarray:
        """Transform (N, 3) coordinates on the host; in and out may alias."""
        src = np.asarray(coords_in)
        if src.ndim != 2 or src.shape[1] != 3:
            raise ValueError(f"coordinates must have shape (N, 3), got {src.shape}")
        moved = (src.astype(np.float64) - self.center) @ self.rotation.rotation_matrix().T \
            + self.center + self.translation
        if coords_out is None:
            return moved.astype(src.dtype if src.dtype.kind == "f" else np.float32)
        dst = coords_out.array if hasattr(coords_out, "array") else np.asarray(coords_out)
        if dst.shape != src.shape:
            raise ValueError(f"output shape {dst.shape} does not match input {src.shape}")
        dst[...] = moved
        return dst

    def inverse(self) -> "Transform":
        """The transform undoing this one, about the same centre."""
        inv = self.rotation.conjugate()
        return Transform(inv, self.center, inv.rotation_matrix() @ (-np.asarray(self.translation)))

    def rotate_vectors(self, vectors) -> np.ndarray:
        """Apply only the rotation (e.g. to gradients): v -> R v, float64."""
        v = np.asarray(vectors, dtype=np.float64)
        return v @ self.rotation.rotation_matrix().T

    def packed(self) -> np.ndarray:
        """15 float64: R row-major (9), center (3), translation (3)."""
        return np.concatenate([self.rotation.rotation_matrix().reshape(9),
                               self.center, self.translation])


def make_transform(center, random_translate=0.0, random_rotation=False, rng=None) -> Transform:
    """Random augmentation about ``center``: SO(3)-uniform rotation when asked,
    then a per-axis uniform translation in [-t, t] when t > 0."""
    center = check_vector3(center, "center")
    t = check_non_negative(random_translate, "random_translate")
    rng = check_rng(rng)
    rot = random_unit_quaternion(rng) if random_rotation else IDENTITY_QUATERNION
    shift = rng.uniform(-t, t, size=3) if t > 0 else np.zeros(3)
    return Transform(rot, center, shift)


def draw_transforms(centers, random_translation, random_rotation, rng) -> list:
    """One ``make_transform`` per example in example order.

    Draws every variate with one ``rng.random((N, k))`` call, which consumes
    the generator stream exactly as N sequential ``make_transform`` calls do
    (each takes 3 rotation then 3 translation doubles; ``uniform(-t, t)`` is
    ``-t + 2t*u``).  ``tests/test_cpu_host.py::test_draw_transforms_matches_sequential_make_transform`` checks the equivalence.
    """
    t = check_non_negative(random_translation, "random_translate")
    centers = np.asarray(centers, dtype=np.float64).reshape(-1, 3)
    n = centers.shape[0]
    k = (3 if random_rotation else 0) + (3 if t > 0 else 0)
    u = rng.random((n, k)) if k else np.zeros((n, 0))
    out = []
    for e in range(n):
        col = 0
        if random_rotation:
            rot = _quaternion_from_uniforms(*u[e, 0:3])
            col = 3
        else:
            rot = IDENTITY_QUATERNION
        if t > 0:
            shift = -t + (2.0 * t) * u[e, col:col + 3]
        else:
            shift = np.zeros(3)
        out.append(Transform(rot, centers[e], shift))
    return out


class TransformArray:
    """A batch of transforms as one (N, 15) float64 array (R row-major,
    center, translation) -- the device format.  Indexing yields ``Transform``
    objects; drawing the array skips per-example object construction."""

    def __init__(self, packed):
        self.packed = np.ascontiguousarray(packed, dtype=np.float64).reshape(-1, 15)

    def __len__(self):
        return self.packed.shape[0]

    def __getitem__(self, e) -> Transform:
        row = self.packed[e]
        return _transform_from_row(row)

    def __iter__(self):
        return (self[e] for e in range(len(self)))


def _transform_from_row(row) -> Transform:
    t = Transform(IDENTITY_QUATERNION, row[9:12], row[12:15])
    object.__setattr__(t, "rotation", _RowRotation(row[:9]))
    return t


class _RowRotation:
    """Rotation given by its matrix (the quaternion is recovered on demand)."""

    def __init__(self, flat):
        self._R = np.array(flat, dtype=np.float64).reshape(3, 3)

    def rotation_matrix(self) -> np.ndarray:
        return self._R.copy()

    def conjugate(self):
        return _RowRotation(self._R.T.reshape(9))

    def rotate(self, vec) -> np.ndarray:
        return self._R @ np.asarray(vec, dtype=np.float64)

    @property
    def angle(self) -> float:
        return math.acos(max(-1.0, min(1.0, (np.trace(self._R) - 1.0) / 2.0)))


def draw_transform_array(centers, random_translation, random_rotation, rng) -> TransformArray:
    """``draw_transforms`` without per-example objects: the same variates and
    the same float64 expressions and libm calls (bit-identical rows), packed
    for the device.  The per-example arithmetic runs in the C ABI helper
    ``gm_draw_transforms``."""
    t = check_non_negative(random_translation, "random_translate")
    centers = np.ascontiguousarray(centers, dtype=np.float64).reshape(-1, 3)
    n = centers.shape[0]
    k = (3 if random_rotation else 0) + (3 if t > 0 else 0)
    u = np.ascontiguousarray(rng.random((n, k))) if k else None
    out = np.empty((n, 15), dtype=np.float64)
    from . import _native

    _native.check(_native.lib().gm_draw_transforms(
        u.ctypes.data if u is not None else None, n, int(bool(random_rotation)), t,
        centers.ctypes.data, out.ctypes.data))
    return TransformArray(out)


def transform_example(t: Transform, example):
    """Apply one transform to every set of an example (coords rounded to f32)."""
    new_sets = [cs.with_coords(t.forward(cs.coords)) for cs in example.coord_sets]
    return type(example)(coord_sets=new_sets, labels=list(example.labels),
                         group=example.group, seqcont=example.seqcont)


# ------------------------------------------------------------------ matmul order
# numpy evaluates (x - c) @ R.T through BLAS; the FMA association of the
# 3-term dot product depends on the BLAS kernel.  The
# device reproduces it to keep binary occupancy bit-exact, so the order is
# probed here once per process.  Codes (shared with csrc/prepare.cu dot3):
#   0..5  fma(a[p2],b[p2], fma(a[p1],b[p1], a[p0]*b[p0])) for permutation p
#   6..8  unfused (a[p0]b[p0] + a[p1]b[p1]) + a[p2]b[p2]
_PERMS = [(0, 1, 2), (1, 0, 2), (0, 2, 1), (2, 0, 1), (1, 2, 0), (2, 1, 0)]
_UNFUSED = [(0, 1, 2), (0, 2, 1), (1, 2, 0)]
_ORDER_CACHE: dict = {}


def _libm_fma():
    libm = ctypes.CDLL(ctypes.util.find_library("m") or "libm.so.6")
    f = libm.fma
    f.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double]
    f.restype = ctypes.c_double
    return f


def _dot_candidates(a, b, fma):
    res = []
    for p in _PERMS:
        res.append(fma(a[p[2]], b[p[2]], fma(a[p[1]], b[p[1]], a[p[0]] * b[p[0]])))
    for p in _UNFUSED:
        res.append((a[p[0]] * b[p[0]] + a[p[1]] * b[p[1]]) + a[p[2]] * b[p[2]])
    return res


def _probe(nrows: int, trials: int, seed: int) -> list:
    fma = _libm_fma()
    rng = np.random.default_rng(seed)
    ok = [True] * (len(_PERMS) + len(_UNFUSED))
    for _ in range(trials):
        q = _quaternion_from_uniforms(*rng.random(3))
        R = q.rotation_matrix()
        c = rng.uniform(-30, 30, 3)
        x = rng.uniform(-60, 60, (nrows, 3)).astype(np.float32).astype(np.float64)
        a = x - c
        got = a @ R.T
        for i in range(nrows):
            for j in range(3):
                cands = _dot_candidates(a[i], R[j], fma)
                for m, v in enumerate(cands):
                    if ok[m] and v != got[i, j]:
                        ok[m] = False
    return [m for m, good in enumerate(ok) if good]


def matmul_order(nrows: int) -> int:
    """Calibrated order code for an (nrows, 3) @ (3, 3) float64 matmul, or -1
    when no candidate reproduces numpy exactly on this host."""
    key = 1 if nrows == 1 else 2
    if key not in _ORDER_CACHE:
        if key == 1:
            good = _probe(1, 400, 11)
        else:
            good = None
            for n, trials in ((2, 60), (3, 40), (17, 8), (300, 1), (1030, 1)):
                g = set(_probe(n, trials, 100 + n))
                good = g if good is None else good & g
            good = sorted(good)
        _ORDER_CACHE[key] = good[0] if good else -1
    return _ORDER_CACHE[key]

"""Kernel input containers: typed coordinate sets and examples.

``CoordinateSet`` keeps the reference's invariants
(/root/reference/pkg/src/voxmol/atomtypes.py:22-96): float32 (N,3) finite
coordinates, float32 positive radii, exactly one of integer ``type_index``
or float32 ``type_vector`` (N,T) >= 0, optional per-type ``type_radii``.
``Example`` mirrors sampling.py:50-61 (only ``coord_sets`` matters for
gridding).  The GridMaker here duck-types its inputs, so the reference's own
``voxmol.CoordinateSet`` / ``voxmol.Example`` objects work unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .validation import check_coords


@dataclass
class CoordinateSet:
    coords: np.ndarray
    radii: np.ndarray
    num_types: int
    type_index: np.ndarray | None = None
    type_vector: np.ndarray | None = None
    type_names: list | None = None
    type_radii: np.ndarray | None = None

    def __post_init__(self):
        self.coords = check_coords(self.coords)
        n = self.coords.shape[0]
        self.radii = np.ascontiguousarray(self.radii, dtype=np.float32).reshape(-1)
        if self.radii.shape[0] != n:
            raise ValueError(f"radii length {self.radii.shape[0]} != atom count {n}")
        if n and not (self.radii > 0).all():
            raise ValueError("all radii must be strictly positive")
        if self.num_types < 1:
            raise ValueError("num_types must be >= 1")
        has_index = self.type_index is not None
        if has_index == (self.type_vector is not None):
            raise ValueError("exactly one of type_index / type_vector must be set")
        if has_index:
            self.type_index = np.ascontiguousarray(self.type_index, dtype=np.int64).reshape(-1)
            if self.type_index.shape[0] != n:
                raise ValueError("type_index length does not match atom count")
            if n and (self.type_index.min() < 0 or self.type_index.max() >= self.num_types):
                raise ValueError(f"type indices must lie in [0, {self.num_types})")
        else:
            self.type_vector = np.ascontiguousarray(self.type_vector, dtype=np.float32)
            if self.type_vector.shape != (n, self.num_types):
                raise ValueError(
                    f"type_vector shape {self.type_vector.shape} != ({n}, {self.num_types})")
            if n and self.type_vector.min() < 0:
                raise ValueError("type_vector components must be >= 0")
        if self.type_radii is not None:
            self.type_radii = np.ascontiguousarray(self.type_radii, dtype=np.float32).reshape(-1)
            if self.type_radii.shape[0] != self.num_types:
                raise ValueError("type_radii length does not match num_types")

    @property
    def num_atoms(self) -> int:
        return int(self.coords.shape[0])

    @property
    def has_vector_types(self) -> bool:
        return self.type_vector is not None

    def centroid(self) -> np.ndarray:
        """float64 mean of the float32 coordinates; origin when empty."""
        if not self.num_atoms:
            return np.zeros(3, dtype=np.float64)
        return self.coords.astype(np.float64).mean(axis=0)

    def with_coords(self, coords) -> "CoordinateSet":
        return CoordinateSet(coords=coords, radii=self.radii, num_types=self.num_types,
                             type_index=self.type_index, type_vector=self.type_vector,
                             type_names=self.type_names, type_radii=self.type_radii)


@dataclass
class Example:
    coord_sets: list
    labels: list = field(default_factory=list)
    group: int | None = None
    seqcont: bool = False

    @property
    def num_coord_sets(self) -> int:
        return len(self.coord_sets)


def make_vector_types(cs) -> CoordinateSet:
    """One-hot ``type_vector`` rows from ``type_index`` (atomtypes.py:294-308)."""
    if cs.type_vector is not None:
        raise ValueError("coordinate set already uses vector types")
    n = cs.coords.shape[0]
    onehot = np.zeros((n, cs.num_types), dtype=np.float32)
    onehot[np.arange(n), cs.type_index] = 1.0
    return CoordinateSet(coords=cs.coords, radii=cs.radii, num_types=cs.num_types,
                         type_vector=onehot, type_names=cs.type_names,
                         type_radii=cs.type_radii)


def coord_sets_of(example) -> list:
    """A lone coordinate set or anything with ``coord_sets`` (voxelizer.py:55-62)."""
    if hasattr(example, "coords") and hasattr(example, "num_types"):
        return [example]
    sets = getattr(example, "coord_sets", None)
    if sets is None:
        raise TypeError(f"cannot voxelize {type(example).__name__}; "
                        "expected a CoordinateSet or an Example")
    return list(sets)


def is_coordinate_set(obj) -> bool:
    return hasattr(obj, "coords") and hasattr(obj, "num_types") and hasattr(obj, "radii")

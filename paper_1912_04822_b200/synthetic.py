"""Synthetic molecules of the benchmark shapes.

Element typing uses the reference's default 14-type element table
(/root/reference/pkg/src/voxmol/atomtypes.py:191-196): channel index and
radius per element.  Typing/parsing itself is out of scope; this module only
produces typed ``CoordinateSet``s of the named shapes:

* ligand: 30 atoms uniform in a 5 A ball, elements C/N/O/S/F/Cl with
  probabilities .70/.10/.14/.02/.02/.02;
* receptor pocket: 1000 atoms uniform in the cube +-15 A, elements C/N/O/S
  with probabilities .62/.17/.19/.02;
* example = [receptor, ligand] -> 28 channels; centre = ligand centroid.

Draw order per example (one generator): receptor coords, receptor elements,
ligand directions, ligand radii, ligand elements (and, for vector typing,
the receptor then ligand weight matrices).
"""

from __future__ import annotations

import numpy as np

from .coordsets import CoordinateSet, Example

TYPE_NAMES = ["C", "N", "O", "S", "P", "F", "Cl", "Br", "I", "B", "Si", "Se", "Metal", "Other"]
TYPE_RADII = np.array([1.90, 1.80, 1.70, 2.00, 2.10, 1.50, 1.80, 2.00, 2.20, 1.92,
                       2.20, 1.90, 1.20, 1.70], dtype=np.float32)
NUM_TYPES = len(TYPE_NAMES)

_LIG_TYPES = np.array([0, 1, 2, 3, 5, 6])
_LIG_P = np.array([0.70, 0.10, 0.14, 0.02, 0.02, 0.02])
_REC_TYPES = np.array([0, 1, 2, 3])
_REC_P = np.array([0.62, 0.17, 0.19, 0.02])

# Rigid offset that mimics PDB frames (SURVEY 8(d) precision probes).
PDB_OFFSET = np.array([41.37, -27.91, 63.05])


def _typed_set(coords, types) -> CoordinateSet:
    types = np.asarray(types, dtype=np.int64)
    return CoordinateSet(coords=np.asarray(coords, dtype=np.float32),
                         radii=TYPE_RADII[types], num_types=NUM_TYPES,
                         type_index=types, type_names=list(TYPE_NAMES),
                         type_radii=TYPE_RADII.copy())


def ligand(rng, n_atoms: int = 30, radius: float = 5.0, offset=None) -> CoordinateSet:
    dirs = rng.standard_normal((n_atoms, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    rad = radius * rng.random(n_atoms) ** (1.0 / 3.0)
    coords = dirs * rad[:, None]
    types = rng.choice(_LIG_TYPES, size=n_atoms, p=_LIG_P)
    if offset is not None:
        coords = coords + offset
    return _typed_set(coords, types)


def receptor(rng, n_atoms: int = 1000, half_width: float = 15.0, offset=None) -> CoordinateSet:
    coords = rng.uniform(-half_width, half_width, (n_atoms, 3))
    types = rng.choice(_REC_TYPES, size=n_atoms, p=_REC_P)
    if offset is not None:
        coords = coords + offset
    return _typed_set(coords, types)


def vectorize(cs: CoordinateSet, rng, density: float = 0.25) -> CoordinateSet:
    """type_vector = U(0,1) * Bernoulli(density) (C4 weights)."""
    w = (rng.random((cs.num_atoms, cs.num_types)) *
         (rng.random((cs.num_atoms, cs.num_types)) < density)).astype(np.float32)
    return CoordinateSet(coords=cs.coords, radii=cs.radii, num_types=cs.num_types,
                         type_vector=w, type_names=cs.type_names, type_radii=cs.type_radii)


def complex_example(rng, n_receptor=1000, n_ligand=30, vector=False, offset=None) -> Example:
    rec = receptor(rng, n_receptor, offset=offset)
    lig = ligand(rng, n_ligand, offset=offset)
    if vector:
        rec = vectorize(rec, rng)
        lig = vectorize(lig, rng)
    return Example(coord_sets=[rec, lig], labels=[1.0])


def batch(n_examples=50, seed=2, n_receptor=1000, n_ligand=30, vector=False,
          offset=None) -> list:
    """C2/C3/C5 (seed 2), C4 (seed 4, vector=True): examples drawn in order."""
    rng = np.random.default_rng(seed)
    return [complex_example(rng, n_receptor, n_ligand, vector, offset)
            for _ in range(n_examples)]


def ligand_only(seed=1, n_atoms=30) -> CoordinateSet:
    """C1: one 30-atom ligand, 14 types."""
    return ligand(np.random.default_rng(seed), n_atoms)

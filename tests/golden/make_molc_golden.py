"""MOLC fixtures from the live reference (build container only):

    python tests/golden/make_molc_golden.py

A cache written by voxmol.chemio.write_cache (chemio.py:242-276) and, per
entry, the CoordinateSet of voxmol.atomtypes.type_molecule(StructureCache.
lookup(name), default_element_typer()) -- coordinates, types, radii."""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from voxmol.atomtypes import default_element_typer, type_molecule  # noqa: E402
from voxmol.chemio import RawAtom, RawMolecule, read_cache, write_cache  # noqa: E402

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "npy")
rng = np.random.default_rng(9)
# common organics, hydrogens / noble gases (dropped silently), metals,
# "other" elements and an unmapped element number (dropped with a warning)
pool = np.array([6] * 12 + [7] * 3 + [8] * 3 + [16, 15, 9, 17, 35, 53, 5, 14, 34, 1, 1, 1, 2,
                 10, 26, 30, 12, 32, 33, 84, 110])
mols = []
for k, n in enumerate([0, 1, 17, 250, 1031]):
    el = rng.choice(pool, size=n)
    xyz = rng.uniform(-20, 60, size=(n, 3)).astype(np.float32)
    mols.append(RawMolecule(name=f"mol{k:02d}_{n}", atoms=[
        RawAtom(int(e), float(x), float(y), float(z)) for e, (x, y, z) in zip(el, xyz)]))
path = os.path.join(HERE, "cache_ref.molc")
write_cache(mols, path)
out = {}
typer = default_element_typer()
with read_cache(path) as c:
    for name in c.names():
        cs = type_molecule(c.lookup(name), typer)
        out[name + "/coords"] = cs.coords
        out[name + "/type_index"] = cs.type_index
        out[name + "/radii"] = cs.radii
np.savez(os.path.join(HERE, "cache_ref_typed.npz"), **out)
print("wrote", path, len(out))

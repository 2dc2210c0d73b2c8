"""Generate golden fixtures by running the LIVE reference (voxmol).

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

It imports ``voxmol`` from /root/reference/pkg/src (read-only, never copied),
feeds it seeded inputs and stores inputs + reference outputs as compressed
``.npz`` files next to this script.  The GPU box never runs this script; the
tests only read the committed fixtures.  ``manifest.json`` records the
versions that produced them (numpy / numba / python), since the reference's
dependencies are unpinned.
"""

from __future__ import annotations

import json
import platform
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))

import numba  # noqa: E402
import voxmol  # noqa: E402
from voxmol.atomtypes import CoordinateSet as RefSet  # noqa: E402
from voxmol.geom import make_transform  # noqa: E402
from voxmol.sampling import Example as RefExample  # noqa: E402
from voxmol.voxelizer import GridMaker as RefGridMaker  # noqa: E402

from paper_1912_04822_b200 import synthetic  # noqa: E402


def rand_set(rng, n, num_types, extent, index_mode=True):
    """Same draw order as the reference fixture random_coordinate_set
    (pkg/tests/conftest.py:63-71)."""
    coords = rng.uniform(-extent, extent, size=(n, 3)).astype(np.float32)
    radii = rng.uniform(1.0, 2.2, size=n).astype(np.float32)
    if index_mode:
        return RefSet(coords=coords, radii=radii, num_types=num_types,
                      type_index=rng.integers(0, num_types, size=n))
    vec = rng.uniform(0.0, 1.0, size=(n, num_types)).astype(np.float32)
    return RefSet(coords=coords, radii=radii, num_types=num_types, type_vector=vec)


def sets_payload(prefix, sets):
    d = {f"{prefix}nsets": np.array(len(sets))}
    for i, cs in enumerate(sets):
        p = f"{prefix}s{i}_"
        d[p + "coords"] = cs.coords
        d[p + "radii"] = cs.radii
        d[p + "num_types"] = np.array(cs.num_types)
        if cs.type_index is not None:
            d[p + "type_index"] = cs.type_index
        else:
            d[p + "type_vector"] = cs.type_vector
        if cs.type_radii is not None:
            d[p + "type_radii"] = cs.type_radii
    return d


def batch_payload(examples):
    d = {"nexamples": np.array(len(examples))}
    for e, ex in enumerate(examples):
        d.update(sets_payload(f"e{e}_", ex.coord_sets))
    return d


def to_ref(cs):
    return RefSet(coords=cs.coords, radii=cs.radii, num_types=cs.num_types,
                  type_index=cs.type_index, type_vector=cs.type_vector,
                  type_radii=cs.type_radii)


def save(name, **arrays):
    path = HERE / f"{name}.npz"
    np.savez_compressed(path, **arrays)
    print(f"{name}: {path.stat().st_size / 1024:.0f} KiB")


def params_payload(gm):
    return {"params": np.array([gm.resolution, gm.dimension, float(gm.binary),
                                float(gm.radius_type_indexed), gm.radius_scale,
                                gm.gaussian_radius_multiple])}


def main():
    # 1. single-set forward, index mode, smooth (cf. test_voxelizer.py:137-146)
    for seed in range(6):
        rng = np.random.default_rng(seed)
        n = int(rng.integers(1, 41))
        cs = rand_set(rng, n, 5, 7.0)
        center = rng.uniform(-1, 1, 3)
        gm = RefGridMaker(dimension=12.0)
        grid = gm.forward(cs, center=center)
        save(f"fwd_index_s{seed}", **sets_payload("", [cs]), center=center, grid=grid,
             **params_payload(gm))

    # 2. parameter variations: radius_scale / grm / odd resolution
    rng = np.random.default_rng(21)
    cs = rand_set(rng, 25, 3, 4.0)
    for tag, kw in (("scale", dict(radius_scale=1.4, gaussian_radius_multiple=1.5, dimension=12.0)),
                    ("res375", dict(resolution=0.375, dimension=9.0)),
                    ("grm05", dict(gaussian_radius_multiple=0.5, dimension=10.0)),
                    ("res03", dict(resolution=0.3, dimension=7.3))):
        gm = RefGridMaker(**kw)
        grid = gm.forward(cs, center=(0.1, -0.2, 0.3))
        save(f"fwd_param_{tag}", **sets_payload("", [cs]), center=np.array([0.1, -0.2, 0.3]),
             grid=grid, **params_payload(gm))

    # 3. batched forward with augmentation, smooth and binary (bit-exact)
    rng = np.random.default_rng(5)
    exs = [RefExample(coord_sets=[rand_set(rng, 60, 4, 6.0), rand_set(rng, 8, 4, 2.5)],
                      labels=[0.0]) for _ in range(4)]
    exs.append(RefExample(coord_sets=[rand_set(rng, 1, 4, 2.0), rand_set(rng, 0, 4, 2.0)],
                          labels=[0.0]))
    for binary in (False, True):
        for tag, aug in (("noaug", dict()),
                         ("rot", dict(random_rotation=True, rng=np.random.default_rng(0))),
                         ("rottr", dict(random_rotation=True, random_translation=2.0,
                                        rng=np.random.default_rng(1))),
                         ("tr", dict(random_translation=1.5, rng=np.random.default_rng(2)))):
            gm = RefGridMaker(dimension=12.0, binary=binary)
            grid = gm.forward_batch(exs, **aug)
            name = f"batch_{'bin' if binary else 'smooth'}_{tag}"
            seed = {"noaug": -1, "rot": 0, "rottr": 1, "tr": 2}[tag]
            extra = dict(aug_seed=np.array(seed),
                         aug_rot=np.array(bool(aug.get("random_rotation", False))),
                         aug_tr=np.array(float(aug.get("random_translation", 0.0))))
            if binary:
                assert set(np.unique(grid)) <= {0.0, 1.0}
                save(name, **batch_payload(exs), bits=np.packbits(grid.reshape(-1) != 0),
                     shape=np.array(grid.shape), **extra, **params_payload(gm))
            else:
                save(name, **batch_payload(exs), grid=grid, **extra, **params_payload(gm))

    # 4. vector mode, radius_type_indexed off/on, smooth and binary
    rng = np.random.default_rng(9)
    vsets = []
    for n in (12, 5):
        s = rand_set(rng, n, 4, 4.0, index_mode=False)
        w = s.type_vector * (rng.random(s.type_vector.shape) < 0.5)
        vsets.append(RefSet(coords=s.coords, radii=s.radii, num_types=4,
                            type_vector=w.astype(np.float32),
                            type_radii=np.array([1.0, 1.5, 2.0, 1.2], np.float32)))
    vex = [RefExample(coord_sets=vsets, labels=[])]
    for rti in (False, True):
        for binary in (False, True):
            gm = RefGridMaker(dimension=10.0, radius_type_indexed=rti, binary=binary)
            grid = gm.forward_batch(vex, random_rotation=True, rng=np.random.default_rng(4))
            save(f"vector_rti{int(rti)}_bin{int(binary)}", **batch_payload(vex), grid=grid,
                 aug_seed=np.array(4), **params_payload(gm))

    # 5. backward, index and vector (per set, explicit center)
    rng = np.random.default_rng(13)
    cs = rand_set(rng, 30, 3, 3.5)
    gm = RefGridMaker(dimension=10.0)
    D = gm.points_per_side()
    gg = rng.standard_normal((3, D, D, D)).astype(np.float32)
    cg, _ = gm.backward(cs, gg, center=(0.2, 0.1, -0.3))
    save("bwd_index", **sets_payload("", [cs]), center=np.array([0.2, 0.1, -0.3]),
         grid_grad=gg, coord_grad=cg, **params_payload(gm))
    for rti in (False, True):
        vs = vsets[0]
        gm = RefGridMaker(dimension=10.0, radius_type_indexed=rti, radius_scale=1.1)
        D = gm.points_per_side()
        gg = np.random.default_rng(14).standard_normal((4, D, D, D)).astype(np.float32)
        cg, tg = gm.backward(vs, gg, center=(0.0, 0.3, 0.1))
        save(f"bwd_vector_rti{int(rti)}", **sets_payload("", [vs]),
             center=np.array([0.0, 0.3, 0.1]), grid_grad=gg, coord_grad=cg, type_grad=tg,
             **params_payload(gm))

    # 6. one C2-shaped example at full size (48^3 x 28), PDB-like offset frame:
    #    smooth forward stored sparse, backward with grid_grad = forward grid,
    #    and the binary grid with augmentation (C3) as packed bits.
    ex = synthetic.batch(1, seed=2, offset=synthetic.PDB_OFFSET)[0]
    rex = RefExample(coord_sets=[to_ref(cs) for cs in ex.coord_sets], labels=[])
    gm = RefGridMaker()
    grid = gm.forward_batch([rex])
    flat = grid.reshape(-1)
    nz = np.flatnonzero(flat).astype(np.int64)
    center = rex.coord_sets[-1].centroid()
    cgs = []
    choff = 0
    for cs in rex.coord_sets:
        cg, _ = gm.backward(cs, grid[0, choff:choff + cs.num_types], center=center)
        cgs.append(cg)
        choff += cs.num_types
    save("c2_example", **batch_payload([rex]), shape=np.array(grid.shape),
         nz_index=nz, nz_value=flat[nz], coord_grad_rec=cgs[0], coord_grad_lig=cgs[1])
    gmb = RefGridMaker(binary=True)
    gridb = gmb.forward_batch([rex, rex], random_rotation=True, random_translation=2.0,
                              rng=np.random.default_rng(0))
    save("c3_example", **batch_payload([rex, rex]), shape=np.array(gridb.shape),
         bits=np.packbits(gridb.reshape(-1) != 0), aug_seed=np.array(0))

    # 7. transforms: numpy's matmul on this host for N=1 and N>=2
    rng = np.random.default_rng(77)
    xs, outs, packs = [], [], []
    for n in (1, 2, 1, 7, 1, 33):
        t = make_transform(rng.uniform(-3, 3, 3), 2.0, True, rng)
        x = rng.uniform(-50, 50, (n, 3)).astype(np.float32)
        xs.append(x)
        outs.append(t.forward(x.astype(np.float64)))
        packs.append(np.concatenate([t.rotation.rotation_matrix().reshape(9), t.center,
                                     t.translation]))
    save("transforms", **{f"x{i}": x for i, x in enumerate(xs)},
         **{f"y{i}": y for i, y in enumerate(outs)}, packs=np.stack(packs))

    manifest = {
        "generator": "tests/golden/make_golden.py",
        "reference": "/root/reference/pkg (voxmol %s)" % voxmol.__version__,
        "python": platform.python_version(),
        "numpy": np.__version__,
        "numba": numba.__version__,
        "machine": platform.machine(),
    }
    (HERE / "manifest.json").write_text(json.dumps(manifest, indent=2) + "\n")


if __name__ == "__main__":
    main()

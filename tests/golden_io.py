"""Load the golden fixtures of tests/golden/ into this package's containers."""

from __future__ import annotations

from pathlib import Path

import numpy as np

from paper_1912_04822_b200.coordsets import CoordinateSet, Example

GOLDEN = Path(__file__).resolve().parent / "golden"


def load(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def sets_from(d: dict, prefix: str = "") -> list:
    out = []
    for i in range(int(d[f"{prefix}nsets"])):
        p = f"{prefix}s{i}_"
        out.append(CoordinateSet(
            coords=d[p + "coords"], radii=d[p + "radii"], num_types=int(d[p + "num_types"]),
            type_index=d.get(p + "type_index"), type_vector=d.get(p + "type_vector"),
            type_radii=d.get(p + "type_radii")))
    return out


def examples_from(d: dict) -> list:
    return [Example(coord_sets=sets_from(d, f"e{e}_"), labels=[])
            for e in range(int(d["nexamples"]))]


def params_from(d: dict) -> dict:
    res, dim, binary, rti, scale, grm = [float(v) for v in d["params"]]
    return dict(resolution=res, dimension=dim, binary=bool(binary),
                radius_type_indexed=bool(rti), radius_scale=scale,
                gaussian_radius_multiple=grm)


def aug_from(d: dict) -> dict:
    seed = int(d.get("aug_seed", -1))
    if seed < 0:
        return {}
    return dict(random_rotation=bool(d.get("aug_rot", True)),
                random_translation=float(d.get("aug_tr", 0.0)),
                rng=np.random.default_rng(seed))


def unpack_bits(d: dict) -> np.ndarray:
    shape = tuple(int(v) for v in d["shape"])
    n = int(np.prod(shape))
    return np.unpackbits(d["bits"])[:n].reshape(shape).astype(np.float32)


def dense_from_sparse(d: dict) -> np.ndarray:
    shape = tuple(int(v) for v in d["shape"])
    flat = np.zeros(int(np.prod(shape)), np.float32)
    flat[d["nz_index"]] = d["nz_value"]
    return flat.reshape(shape)


BATCH_FIXTURES = [f"batch_{m}_{a}" for m in ("smooth", "bin")
                  for a in ("noaug", "rot", "rottr", "tr")]
VECTOR_FIXTURES = [f"vector_rti{r}_bin{b}" for r in (0, 1) for b in (0, 1)]
SINGLE_FIXTURES = [f"fwd_index_s{s}" for s in range(6)] + \
    [f"fwd_param_{t}" for t in ("scale", "res375", "grm05", "res03")]


def expected_grid(d: dict) -> np.ndarray:
    return unpack_bits(d) if "bits" in d else d["grid"]

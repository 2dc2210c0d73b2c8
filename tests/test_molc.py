"""MOLC cache -> typed atoms against the reference's own
reader + typer outputs (tests/golden/make_molc_golden.py)."""
from pathlib import Path

import numpy as np
import pytest

NPY = Path(__file__).resolve().parent / "golden" / "npy"


def _ref():
    z = np.load(NPY / "cache_ref_typed.npz")
    names = sorted({k.split("/")[0] for k in z.files})
    return z, names


def test_typed_matches_reference_type_molecule():
    from paper_1912_04822_b200.molc import MolcCache

    z, names = _ref()
    with MolcCache(NPY / "cache_ref.molc") as c:
        assert c.names() == names and len(c) == len(names)
        for n in names:
            cs = c.typed(n)
            np.testing.assert_array_equal(cs.coords, z[n + "/coords"])
            np.testing.assert_array_equal(cs.type_index, z[n + "/type_index"])
            np.testing.assert_array_equal(cs.radii, z[n + "/radii"])
            assert cs.num_types == 14


def test_write_molc_roundtrip_bytes(tmp_path):
    """Our writer reproduces the reference file byte for byte."""
    from paper_1912_04822_b200.molc import MolcCache, write_molc

    with MolcCache(NPY / "cache_ref.molc") as c:
        mols = []
        for n in sorted(c._index, key=c._index.get):  # file (insertion) order
            r = c.records(n)
            mols.append((n, r["element"], np.stack([r["x"], r["y"], r["z"]], 1)))
    out = tmp_path / "c.molc"
    write_molc(mols, out)
    assert out.read_bytes() == (NPY / "cache_ref.molc").read_bytes()


def test_molc_errors(tmp_path):
    from paper_1912_04822_b200 import FormatError
    from paper_1912_04822_b200.molc import MolcCache

    bad = tmp_path / "bad.molc"
    bad.write_bytes(b"XXXX" + b"\0" * 40)
    with pytest.raises(FormatError):
        MolcCache(bad)
    good = (NPY / "cache_ref.molc").read_bytes()
    cut = tmp_path / "cut.molc"
    cut.write_bytes(good[:-3])
    with pytest.raises(FormatError):
        MolcCache(cut)
    with MolcCache(NPY / "cache_ref.molc") as c:
        with pytest.raises(KeyError):
            c.typed("missing")


@pytest.mark.gpu
def test_to_device_matches_reference():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1912_04822_b200.molc import MolcCache

    z, names = _ref()
    with MolcCache(NPY / "cache_ref.molc") as c:
        d = c.to_device(names)
    off = d["offsets"].cpu().numpy()
    for e, n in enumerate(names):
        s = slice(off[e], off[e + 1])
        np.testing.assert_array_equal(d["coords"][s].cpu().numpy(), z[n + "/coords"])
        np.testing.assert_array_equal(d["type_index"][s].cpu().numpy(), z[n + "/type_index"])
        np.testing.assert_array_equal(d["radius"][s].cpu().numpy(), z[n + "/radii"])


@pytest.mark.gpu
def test_device_decode_many_entries_vs_host_typing(tmp_path):
    """gm_molc_decode over 1500 entries (several scan chunks), entries longer
    than one 256-atom chunk, empty entries and entries whose atoms are all
    dropped (hydrogens): equal to the host typing (pinned to the reference's
    type_molecule above), entry by entry."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1912_04822_b200.molc import MolcCache, write_molc

    rng = np.random.default_rng(3)
    elements = np.array([1, 1, 6, 6, 6, 7, 8, 16, 15, 9, 17, 35, 53, 5, 14, 34, 26, 2, 10, 33, 0, 200])
    mols = []
    for k in range(1500):
        n = int(rng.choice([0, 1, 3, 40, 255, 256, 257, 700]))
        el = rng.choice(elements, n).astype(np.uint8)
        if k % 97 == 0:
            el[:] = 1  # hydrogens only: every atom dropped
        mols.append((f"m{k:05d}", el, rng.normal(0, 20, (n, 3)).astype(np.float32)))
    path = tmp_path / "many.molc"
    write_molc(mols, path)
    with MolcCache(path) as c:
        names = [f"m{k:05d}" for k in rng.permutation(1500)]
        d = c.to_device(names)
        off = d["offsets"].cpu().numpy()
        coords, ti, rad = (d[k].cpu().numpy() for k in ("coords", "type_index", "radius"))
        assert off[0] == 0 and off[-1] == coords.shape[0]
        for e, n in enumerate(names):
            cs = c.typed(n)
            s = slice(off[e], off[e + 1])
            np.testing.assert_array_equal(coords[s], cs.coords)
            np.testing.assert_array_equal(ti[s], cs.type_index)
            np.testing.assert_array_equal(rad[s], cs.radii)
        empty = c.to_device([])
        assert empty["offsets"].cpu().tolist() == [0] and empty["coords"].shape[0] == 0

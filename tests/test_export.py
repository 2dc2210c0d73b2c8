"""NPY + JSON sidecar export against fixtures written by
the live reference (tests/golden/make_npy_golden.py): byte-identical files."""
from pathlib import Path

import numpy as np
import pytest

NPY = Path(__file__).resolve().parent / "golden" / "npy"
CASES = ["vec_f32", "grid_f32", "grid_f64", "big_header"]


@pytest.mark.parametrize("name", CASES)
def test_write_npy_bytes_match_reference(name, tmp_path):
    from paper_1912_04822_b200.export import read_npy, write_npy

    arr = np.load(NPY / f"{name}_input.npy")
    out = tmp_path / "x.npy"
    write_npy(out, arr)
    assert out.read_bytes() == (NPY / f"{name}_ref.npy").read_bytes()
    np.testing.assert_array_equal(read_npy(NPY / f"{name}_ref.npy"), arr)


def test_save_grid_matches_reference(tmp_path):
    from paper_1912_04822_b200 import save_grid

    arr = np.load(NPY / "grid_f32_input.npy")
    side = save_grid(tmp_path / "saved.npy", arr,
                     origin=np.array([[-11.75, -11.75, -11.75], [1.0, 2.0, 3.0]]),
                     resolution=0.5, channel_labels=[f"rec:{i}" for i in range(3)],
                     extra={"note": "fixture"})
    assert Path(side).name == "saved.json"
    assert (tmp_path / "saved.npy").read_bytes() == (NPY / "saved_ref.npy").read_bytes()
    assert Path(side).read_text() == (NPY / "saved_ref.json").read_text()


def test_read_npy_errors(tmp_path):
    from paper_1912_04822_b200 import FormatError
    from paper_1912_04822_b200.export import read_npy

    bad = tmp_path / "bad.npy"
    bad.write_bytes(b"NOTNPY" + b"\0" * 20)
    with pytest.raises(FormatError):
        read_npy(bad)
    good = (NPY / "grid_f32_ref.npy").read_bytes()
    trunc = tmp_path / "trunc.npy"
    trunc.write_bytes(good[:-8])
    with pytest.raises(FormatError):
        read_npy(trunc)
    with pytest.raises(TypeError):
        from paper_1912_04822_b200.export import write_npy
        write_npy(tmp_path / "i.npy", np.zeros(3, np.int32))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["grid_f32", "big_header", "grid_f64"])
def test_write_npy_streams_device_tensors(name, tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1912_04822_b200.export import write_npy

    t = torch.from_numpy(np.load(NPY / f"{name}_input.npy")).cuda()
    out = tmp_path / "d.npy"
    write_npy(out, t, chunk_bytes=1000)  # many chunks through both pinned buffers
    assert out.read_bytes() == (NPY / f"{name}_ref.npy").read_bytes()

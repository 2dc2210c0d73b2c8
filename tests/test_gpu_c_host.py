"""The C ABI from a non-Python host: tests/c_host/c_host_test.c packs a batch
by hand, drives gm_prepare_inline -> gm_forward -> gm_backward with its own
device buffers, and checks the results against the C oracle (exit 0 =
parity within 1e-6 abs + 1e-5 rel).  Compiled here with gcc against the
in-tree library, the oracle and the CUDA runtime."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CUDA = Path("/usr/local/cuda")


@pytest.mark.gpu
def test_c_host_drives_the_abi(tmp_path):
    lib = ROOT / "paper_1912_04822_b200"
    if not (lib / "libgridmaker_b200.so").exists() or not (ROOT / "oracle" / "liboracle.so").exists():
        pytest.skip("libraries not built")
    exe = tmp_path / "c_host_test"
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", str(ROOT / "tests" / "c_host" / "c_host_test.c"),
           f"-I{ROOT / 'include'}", f"-I{CUDA / 'include'}", f"-L{lib}", "-lgridmaker_b200",
           f"-L{ROOT / 'oracle'}", "-loracle", f"-L{CUDA / 'lib64'}", "-lcudart", "-lm",
           f"-Wl,-rpath,{lib}:{ROOT / 'oracle'}:{CUDA / 'lib64'}", "-o", str(exe)]
    build = subprocess.run(cmd, capture_output=True, text=True)
    assert build.returncode == 0, build.stderr
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    print(run.stdout)
    assert run.returncode == 0, run.stdout + run.stderr
    assert "0 bad" in run.stdout

"""The reference's OWN hot-path test files, unmodified, run on the GPU against
this implementation ("the reference suite as the drop-in
acceptance harness").

``tests/_refsuite.tar.gz`` (made by tools/vendor_refsuite.py in the build
container, git-ignored) holds /root/reference/pkg/src/voxmol and
pkg/tests/{conftest,oracles,test_voxelizer,test_geom,test_acceptance}.py
byte for byte, with their SHA-256 digests.  Each case unpacks it into a
temporary directory, re-checks the digests and runs pytest on one reference
file in a subprocess with ``-p refsuite_plugin``:

* ``kernels``: the reference's host code calls our sm_100a kernels through
  ``paper_1912_04822_b200.kernels`` substituted for ``voxmol._kernels`` (the
  one-line switch of INTEGRATION.md section 1);
* ``gridmaker``: ``voxmol.voxelizer.GridMaker`` is our ``GridMaker``.

Deselected, with the reason: ``test_acceptance.py::test_determinism_under_parallelism``
(it times the reference's numba CPU thread scaling, >= 3x on 8+ host threads,
and re-runs the CLI in subprocesses -- a property of the CPU backend, not of
the gridding path).  ``test_sampler_distribution`` and
``test_grouped_sequences`` run (they do not grid; the sampler is the
reference's own).
"""

import hashlib
import json
import os
import subprocess
import sys
import tarfile
from pathlib import Path

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
ARCHIVE = HERE / "_refsuite.tar.gz"
DESELECT = {"test_acceptance.py": ["test_determinism_under_parallelism"]}


@pytest.fixture(scope="module")
def suite(tmp_path_factory):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not ARCHIVE.exists():
        pytest.skip("tests/_refsuite.tar.gz missing (run tools/vendor_refsuite.py where "
                    "/root/reference exists)")
    d = tmp_path_factory.mktemp("refsuite")
    with tarfile.open(ARCHIVE) as tar:
        tar.extractall(d, filter="data")
    man = json.loads((d / "MANIFEST.json").read_text())
    for rel, digest in man["files"].items():
        assert hashlib.sha256((d / rel).read_bytes()).hexdigest() == digest, f"{rel} was modified"
    return d


@pytest.mark.parametrize("mode", ["kernels", "gridmaker"])
@pytest.mark.parametrize("name", ["test_voxelizer.py", "test_geom.py", "test_acceptance.py"])
def test_reference_suite(suite, mode, name):
    env = dict(os.environ)
    env["GM_REFSUITE_MODE"] = mode
    env["PYTHONPATH"] = os.pathsep.join([str(suite / "src"), str(HERE), str(ROOT),
                                         env.get("PYTHONPATH", "")])
    args = [sys.executable, "-m", "pytest", "-p", "refsuite_plugin", "-q", "-rA",
            "-p", "no:cacheprovider", str(suite / "tests" / name)]
    if DESELECT.get(name):
        args += ["-k", " and ".join(f"not {t}" for t in DESELECT[name])]
    r = subprocess.run(args, cwd=str(suite / "tests"), env=env, capture_output=True, text=True,
                       timeout=1800)
    log = ROOT / "gpurun_out"
    if log.is_dir():
        (log / f"refsuite_{mode}_{name}.txt").write_text(r.stdout + "\n" + r.stderr)
    tail = "\n".join(r.stdout.strip().splitlines()[-25:])
    assert r.returncode == 0, f"reference {name} ({mode}) failed:\n{tail}\n{r.stderr[-2000:]}"
    passed = [ln for ln in r.stdout.splitlines() if ln.startswith("PASSED")]
    assert passed, tail
    assert "failed" not in r.stdout.splitlines()[-1], tail

#!/usr/bin/env python
"""Pack the reference's hot-path test files and its package, UNMODIFIED, into
``tests/_refsuite.tar.gz`` (a git-ignored test fixture, not product source)
so the GPU box -- where /root/reference does not exist -- can run them against
this implementation through ``tests/refsuite_plugin.py``.  The archive is
unpacked into a temporary directory at test time only.

Copied: ``pkg/src/voxmol/*.py`` (the reference package, needed by its own
tests) and ``pkg/tests/{conftest,oracles,test_voxelizer,test_geom,
test_acceptance}.py``.  A manifest of SHA-256 digests of the sources is
stored in the archive; ``tests/test_gpu_refsuite.py`` re-hashes the
unpacked files before running them, so an edited copy fails loudly.

Runs from ``__graft_entry__.build()`` whenever /root/reference is present.
"""

from __future__ import annotations

import hashlib
import io
import json
import sys
import tarfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/pkg")
DEST = ROOT / "tests" / "_refsuite.tar.gz"
TESTS = ["conftest.py", "oracles.py", "test_voxelizer.py", "test_geom.py", "test_acceptance.py"]


def sha256(p: Path) -> str:
    return hashlib.sha256(p.read_bytes()).hexdigest()


def main() -> int:
    if not (REF / "src" / "voxmol").is_dir():
        print(f"vendor_refsuite: {REF} not present, nothing to do")
        return 0
    files = [(f, f"src/voxmol/{f.name}") for f in sorted((REF / "src" / "voxmol").glob("*.py"))]
    files += [(REF / "tests" / n, f"tests/{n}") for n in TESTS]
    manifest = {arc: sha256(f) for f, arc in files}
    tmp = DEST.with_suffix(".tmp")
    with tarfile.open(tmp, "w:gz") as tar:
        for f, arc in files:
            tar.add(f, arcname=arc)
        data = json.dumps({"source": str(REF), "files": manifest}, indent=1,
                          sort_keys=True).encode()
        info = tarfile.TarInfo("MANIFEST.json")
        info.size = len(data)
        tar.addfile(info, io.BytesIO(data))
    tmp.replace(DEST)
    print(f"vendor_refsuite: {len(files)} files -> {DEST}")
    return 0


if __name__ == "__main__":
    sys.exit(main())

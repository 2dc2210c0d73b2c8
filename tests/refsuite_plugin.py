"""pytest plugin: run the reference's own test files against this
implementation (loaded with ``-p refsuite_plugin`` by test_gpu_refsuite.py).

``GM_REFSUITE_MODE``:

* ``kernels`` -- the INTEGRATION.md section 1 switch: ``voxmol._kernels`` (the
  numba kernel module /root/reference/pkg/src/voxmol/_kernels.py) is replaced by
  ``paper_1912_04822_b200.kernels`` before ``voxmol.voxelizer`` imports it.  The
  reference's host code (validation, packing, transforms) then calls the
  sm_100a kernels through the C ABI's ``*_host`` entry points.
* ``gridmaker`` -- the reference's ``GridMaker`` class is replaced by
  ``paper_1912_04822_b200.GridMaker`` (the whole host + device path), before
  any test module does ``from voxmol.voxelizer import GridMaker``; the kernel
  module is swapped too, so numba never compiles anything.
"""

import os
import sys


def _install():
    mode = os.environ.get("GM_REFSUITE_MODE", "kernels")
    from paper_1912_04822_b200 import kernels as gpu_kernels

    sys.modules["voxmol._kernels"] = gpu_kernels
    import voxmol

    voxmol._kernels = gpu_kernels
    if mode == "gridmaker":
        import voxmol.errors
        import voxmol.voxelizer as vz
        from paper_1912_04822_b200 import GridMaker, errors

        errors.use_exception_classes(voxmol.errors)  # callers catch voxmol's classes

        vz.GridMaker = GridMaker
        voxmol.GridMaker = GridMaker
    elif mode != "kernels":
        raise RuntimeError(f"unknown GM_REFSUITE_MODE {mode!r}")
    import voxmol.voxelizer as vz2

    assert vz2._kernels is gpu_kernels, "the reference voxelizer still binds numba kernels"


def pytest_configure(config):
    _install()


def pytest_report_header(config):
    return f"refsuite: voxmol._kernels -> paper_1912_04822_b200.kernels " \
           f"(mode {os.environ.get('GM_REFSUITE_MODE', 'kernels')})"

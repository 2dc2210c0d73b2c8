"""Exception types of the gridding path.

Mirrors the classes the reference raises on this path
(/root/reference/pkg/src/voxmol/errors.py:4-33): ``ConfigError`` is raised by
``GridMaker`` for ``radius_type_indexed`` without a radius table
(voxelizer.py:315); ``FormatError`` by the MOLC / NPY readers.  ``DeviceError`` is ours: a CUDA launch/resource failure
reported through the C ABI status code.
"""


class VoxmolError(Exception):
    """Base class of gridding failures."""


class ConfigError(VoxmolError, ValueError):
    """Options are inconsistent with each other or with the data."""


class FormatError(VoxmolError, ValueError):
    """A binary container (MOLC cache, NPY file) is malformed or truncated
    (errors.py:28-29)."""


class DeviceError(VoxmolError, RuntimeError):
    """The CUDA extension reported a launch or resource failure."""


def use_exception_classes(ref_errors) -> None:
    """Raise the reference's own exception classes from now on.

    For mixed deployments where callers catch ``voxmol.errors.ConfigError``
    / ``FormatError`` (e.g. the reference's test suite run against this
    GridMaker, tests/refsuite_plugin.py): pass the reference's ``errors``
    module and every raise site of this package (which looks the class up
    in this module at raise time) uses its classes.
    """
    g = globals()
    for name in ("VoxmolError", "ConfigError", "FormatError"):
        if hasattr(ref_errors, name):
            g[name] = getattr(ref_errors, name)

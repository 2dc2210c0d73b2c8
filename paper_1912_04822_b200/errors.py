"""Exception types of the gridding path.

Mirrors the classes the reference raises on this path
(/root/reference/pkg/src/voxmol/errors.py:4-33): ``ConfigError`` is raised by
``GridMaker`` for ``radius_type_indexed`` without a radius table
(voxelizer.py:315).  ``DeviceError`` is ours: a CUDA launch/resource failure
reported through the C ABI status code.
"""


class VoxmolError(Exception):
    """Base class of gridding failures."""


class ConfigError(VoxmolError, ValueError):
    """Options are inconsistent with each other or with the data."""


class DeviceError(VoxmolError, RuntimeError):
    """The CUDA extension reported a launch or resource failure."""

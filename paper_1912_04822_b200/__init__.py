"""B200-native GridMaker hot path of libmolgrid (arXiv 1912.04822).

Drop-in for the gridding path of the reference ``voxmol`` package:
``GridMaker`` (forward / forward_batch / backward, plus backward_batch and
device-resident packed batches), the rigid ``Transform`` augmentation, and
the ``CoordinateSet`` / ``Example`` containers.  All arithmetic runs in the
in-tree CUDA extension (``libgridmaker_b200.so``, sm_100a) via its C ABI.
"""

from .coordsets import CoordinateSet, Example, make_vector_types
from .dataset import AssembledBatch, DeviceDataset
from .errors import ConfigError, DeviceError, FormatError, VoxmolError
from .export import read_npy, write_npy
from .geom import (IDENTITY_QUATERNION, Quaternion, Transform, draw_transforms,
                   make_transform, random_unit_quaternion, transform_example)
from .graph import GraphStep
from .pipeline import DatasetBatches, DeviceBatchPipeline
from .grids import GridShape, GridView, OwnedGrid, copy_into, make_grid, view_over
from .voxelizer import (GridMaker, channel_count, channel_names, get_num_threads, save_grid,
                        set_num_threads)

__version__ = "0.1.0"

__all__ = [
    "CoordinateSet", "Example", "make_vector_types", "ConfigError", "DeviceError",
    "VoxmolError", "FormatError", "read_npy", "write_npy", "IDENTITY_QUATERNION", "Quaternion", "Transform", "draw_transforms",
    "make_transform", "random_unit_quaternion", "transform_example", "GridMaker",
    "channel_count", "channel_names", "save_grid", "set_num_threads", "get_num_threads", "GraphStep",
    "GridShape", "GridView", "OwnedGrid", "copy_into", "make_grid", "view_over",
    "DeviceDataset", "AssembledBatch", "DatasetBatches", "DeviceBatchPipeline",
]

"""Small end-to-end run of every kernel family (a crash / illegal-address check):
host-packed and device-assembled batches (index and vector typing, smooth
and binary, 48^3 / 96^3 / odd grids), the reference-shaped kernels module."""
import sys

sys.path.insert(0, "/root/repo")
import numpy as np
import torch

from paper_1912_04822_b200 import GridMaker, geom, kernels, synthetic
from paper_1912_04822_b200.dataset import DeviceDataset

rng = np.random.default_rng(0)
for vector in (False, True):
    exs = synthetic.batch(4, seed=2, vector=vector)
    ds = DeviceDataset(exs)
    for cfg in (dict(), dict(binary=True), dict(resolution=0.25, dimension=23.75),
                dict(resolution=0.375, dimension=9.0, radius_type_indexed=vector)):
        gm = GridMaker(**cfg)
        for pb in (gm.pack(exs), ds.batch(4).assemble(gm, [3, 1, 0, 2])):
            xf = geom.draw_transform_array(pb.default_centers, 2.0, True, rng)
            out, _ = gm.forward_packed(pb, transforms=xf)
            gm.backward_packed(pb, out.clone(), reuse_prepared=True)
            gm.backward_packed(pb, out.clone(), transforms=xf)
        torch.cuda.synchronize()
    g = GridMaker().forward_batch(exs[:2], random_rotation=True, rng=rng)
    GridMaker().backward_batch(exs[:2], g)
cs = exs[0].coord_sets[0]
origin = GridMaker().grid_origin(cs.centroid())
gg = np.random.default_rng(1).standard_normal((14, 48, 48, 48)).astype(np.float32)
kernels.backward_vector(cs.coords.astype(np.float64), cs.radii.astype(np.float64),
                        cs.type_vector.astype(np.float64), gg, np.ones(14), False, origin,
                        0.5, 1.0, 1.5)
torch.cuda.synchronize()
print("sanitize smoke ok")

"""k_prepare_static duration vs batch size (run under ncu --metrics gpu__time_duration.sum)."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import torch
from paper_1912_04822_b200 import GridMaker, geom, synthetic

gm = GridMaker()
for n in (1, 8, 9, 50, 64, 65, 200):
    exs = synthetic.batch(n, seed=2)
    pb = gm.pack(exs)
    xf = geom.draw_transform_array(pb.default_centers, 2.0, True, np.random.default_rng(0))
    for _ in range(3):
        gm._prepare(pb, None, xf, 48)
    torch.cuda.synchronize()

"""gm_prepare_inline device time (CUDA events) on the bench configs."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import torch
import bench
from paper_1912_04822_b200 import GridMaker, geom

for name in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["c2"]):
    cfg = bench.CONFIGS[name]
    exs, centers = bench.make_batch(cfg, 0, 1)
    gm = GridMaker(resolution=cfg["resolution"], dimension=cfg["dimension"], binary=cfg["binary"])
    pb = gm.pack(exs)
    D = gm.points_per_side()
    xf = geom.draw_transform_array(pb.default_centers, 2.0, True, np.random.default_rng(0))
    for _ in range(5):
        gm._prepare(pb, None, xf, D)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 200
    a.record()
    for _ in range(n):
        gm._prepare(pb, None, xf, D)
    b.record()
    torch.cuda.synchronize()
    print(f"{name} prepare {a.elapsed_time(b) / n * 1e3:8.1f} us (includes host launch rate)")

"""Device time of the packed C2 step pieces (CUDA events around prepare, forward, backward)."""
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
    out = torch.empty((pb.nexamples, pb.nchannels, D, D, D), device="cuda")
    gg = torch.randn_like(out)
    rng = np.random.default_rng(0)
    def step():
        gm.forward_packed(pb, out, transforms=geom.draw_transform_array(pb.default_centers, 2.0, True, rng))
        gm.backward_packed(pb, gg, reuse_prepared=True)
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 50
    a.record()
    for _ in range(n):
        step()
    b.record()
    torch.cuda.synchronize()
    print(f"{name} step {a.elapsed_time(b) / n * 1e3:8.1f} us")

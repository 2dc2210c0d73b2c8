"""Eager packed step vs GraphStep replay: wall time per call (host-issue bound
for small batches) and device time, for the bench configs named in argv[1]."""
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np
import torch

import bench
from paper_1912_04822_b200 import GridMaker, geom

for name in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["c1", "c2"]):
    cfg = bench.CONFIGS[name]
    exs, centers = bench.make_batch(cfg, 0, 1)
    gm = GridMaker(resolution=cfg["resolution"], dimension=cfg["dimension"], binary=cfg["binary"])
    pb = gm.pack(exs)
    D = gm.points_per_side()
    out = torch.empty((pb.nexamples, pb.nchannels, D, D, D), device="cuda")
    gg = torch.randn_like(out)
    rng = np.random.default_rng(0)
    step = gm.capture_step(pb, backward=True, grid_grad=gg)

    def eager():
        xf = geom.draw_transform_array(pb.default_centers, 2.0, True, rng)
        gm.forward_packed(pb, out, transforms=xf)
        gm.backward_packed(pb, gg, reuse_prepared=True)

    def graph():
        step.run(random_rotation=True, random_translation=2.0, rng=rng)

    for label, fn in (("eager", eager), ("graph", graph), ("eager", eager), ("graph", graph)):
        for _ in range(10):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 200 if pb.nexamples < 8 else 50
        t0 = time.perf_counter()
        a.record()
        for _ in range(n):
            fn()
        t1 = time.perf_counter()
        b.record()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"{name} {label}: host issue {(t1 - t0) / n * 1e6:7.1f} us/call, "
              f"wall {(t2 - t0) / n * 1e6:7.1f} us/call, device {a.elapsed_time(b) / n * 1e3:7.1f} us/call")

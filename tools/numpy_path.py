"""Where the numpy (reference-shaped) path spends its time on C2: host packing,
gridding, device->host of the grids (pageable vs pinned), host->device of a
numpy grid_grad, backward."""
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np
import torch

import bench
from paper_1912_04822_b200 import GridMaker, geom

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
exs, _ = bench.make_batch(cfg, 0, 1)
gm = GridMaker(resolution=cfg["resolution"], dimension=cfg["dimension"], binary=cfg["binary"])
rng = np.random.default_rng(0)


def t(label, fn, n=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        r = fn()
    torch.cuda.synchronize()
    print(f"{label:40s} {(time.perf_counter() - t0) / n * 1e3:8.2f} ms")
    return r


sets = [ex.coord_sets for ex in exs]
pb = t("pack", lambda: gm.pack(sets))
D = gm.points_per_side()
dout = torch.empty((pb.nexamples, pb.nchannels, D, D, D), device="cuda")
t("forward_packed", lambda: gm.forward_packed(pb, dout, random_rotation=True,
                                              random_translation=2.0, rng=rng))
t("d2h .cpu() (pageable, fresh)", lambda: dout.cpu())
pin = torch.empty(dout.shape, dtype=torch.float32, pin_memory=True)
t("d2h into pinned (reused)", lambda: pin.copy_(dout))
t("d2h into fresh pinned (cached alloc)",
  lambda: torch.empty(dout.shape, dtype=torch.float32, pin_memory=True).copy_(dout))
host = dout.cpu().numpy()
t("np.empty + copy (page faults)", lambda: np.copyto(np.empty_like(host), host))
t("h2d from pageable numpy", lambda: torch.from_numpy(host).to("cuda"))
t("h2d from pinned", lambda: pin.to("cuda"))
gg = torch.from_numpy(host).to("cuda")
t("backward_packed", lambda: gm.backward_packed(pb, gg, reuse_prepared=True))
t("forward_batch (numpy)", lambda: gm.forward_batch(exs, random_rotation=True,
                                                    random_translation=2.0, rng=rng))
t("backward_batch (numpy grad)", lambda: gm.backward_batch(exs, host))

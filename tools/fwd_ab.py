"""A/B of library builds (GM_LIB selects the .so): per config, the forward
grid's SHA-256 (bitwise comparison across builds), the backward gradients'
SHA-256, and device times of forward / backward / step (CUDA events).
usage: [GM_LIB=...] python tools/fwd_ab.py c2,c4,c5"""
import hashlib
import os
import sys

sys.path.insert(0, "/root/repo")
import numpy as np
import torch

import bench
from paper_1912_04822_b200 import GridMaker, geom

tag = os.path.basename(os.environ.get("GM_LIB", "default"))
for name in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["c2"]):
    cfg = bench.CONFIGS[name]
    exs, centers = bench.make_batch(cfg, 0, 1)
    gm = GridMaker(resolution=cfg["resolution"], dimension=cfg["dimension"], binary=cfg["binary"])
    pb = gm.pack(exs)
    D = gm.points_per_side()
    out = torch.empty((pb.nexamples, pb.nchannels, D, D, D), device="cuda")
    gg = torch.randn(out.shape, generator=torch.Generator(device="cuda").manual_seed(7),
                     device="cuda")
    tg = torch.empty(max(pb.nweights, 1), device="cuda") if pb.vector_mode else None
    xf = geom.draw_transform_array(pb.default_centers, 2.0, True, np.random.default_rng(0))
    gm.forward_packed(pb, out, transforms=xf)
    cg, tgo = gm.backward_packed(pb, gg, reuse_prepared=True, type_grad=tg)
    torch.cuda.synchronize()
    h1 = hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()[:16]
    h2 = hashlib.sha256(cg.cpu().numpy().tobytes()).hexdigest()[:16]
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    n = 30
    fe = [(ev(), ev()) for _ in range(n)]
    be = [(ev(), ev()) for _ in range(n)]
    for k in range(n):
        gm.forward_packed(pb, out, transforms=xf, events=fe[k])
        gm.backward_packed(pb, gg, reuse_prepared=True, type_grad=tg, events=be[k])
    a, b = ev(), ev()
    a.record()
    for k in range(n):
        gm.forward_packed(pb, out, transforms=xf)
        gm.backward_packed(pb, gg, reuse_prepared=True, type_grad=tg)
    b.record()
    torch.cuda.synchronize()
    f = np.median([x.elapsed_time(y) for x, y in fe]) * 1e3
    bw = np.median([x.elapsed_time(y) for x, y in be]) * 1e3
    print(f"{tag:24s} {name} fwd {f:7.1f} us  bwd {bw:7.1f} us  step "
          f"{a.elapsed_time(b) / n * 1e3:7.1f} us  grid {h1} grad {h2}")

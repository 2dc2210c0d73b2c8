"""Host-side cost per step of the packed fwd+bwd calls vs device time."""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import torch
from paper_1912_04822_b200 import GridMaker, geom, synthetic

exs = synthetic.batch(50, seed=2)
gm = GridMaker()
pb = gm.pack(exs)
out = torch.empty((50, 28, 48, 48, 48), device="cuda")
gg = torch.randn_like(out)
cg = torch.empty((pb.natoms, 3), device="cuda")
rng = np.random.default_rng(0)
centers = pb.default_centers
for _ in range(5):
    gm.forward_packed(pb, out, transforms=geom.draw_transform_array(centers, 2.0, True, rng))
    gm.backward_packed(pb, gg, reuse_prepared=True, coord_grad=cg)
torch.cuda.synchronize()
for label, fn in (("draw", lambda: geom.draw_transform_array(centers, 2.0, True, rng)),):
    t = time.perf_counter()
    for _ in range(200):
        fn()
    print(label, (time.perf_counter() - t) / 200 * 1e6, "us")
t0 = time.perf_counter()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    gm.forward_packed(pb, out, transforms=geom.draw_transform_array(centers, 2.0, True, rng))
    gm.backward_packed(pb, gg, reuse_prepared=True, coord_grad=cg)
t1 = time.perf_counter()
e1.record()
torch.cuda.synchronize()
t2 = time.perf_counter()
print("host issue per step", (t1 - t0) / 50 * 1e6, "us; device per step", e0.elapsed_time(e1) / 50 * 1e3, "us; wall", (t2 - t0) / 50 * 1e6)
# the same loop with one fixed transform array (no per-step draw)
xf = geom.draw_transform_array(centers, 2.0, True, rng)
torch.cuda.synchronize()
t0 = time.perf_counter()
e0.record()
for _ in range(50):
    gm.forward_packed(pb, out, transforms=xf)
    gm.backward_packed(pb, gg, reuse_prepared=True, coord_grad=cg)
t1 = time.perf_counter()
e1.record()
torch.cuda.synchronize()
print("fixed xf: host issue per step", (t1 - t0) / 50 * 1e6, "us; device per step",
      e0.elapsed_time(e1) / 50 * 1e3, "us")

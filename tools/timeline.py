"""Per-step device timeline of the C2 bench step (events between the pieces)."""
import ctypes
import sys

sys.path.insert(0, "/root/repo")
import numpy as np
import torch

from paper_1912_04822_b200 import GridMaker, _native, geom, synthetic
from paper_1912_04822_b200.voxelizer import stream_handle

exs = synthetic.batch(50, seed=2)
gm = GridMaker()
pb = gm.pack(exs)
D = gm.points_per_side()
out = torch.empty((50, 28, D, D, D), device="cuda")
gg = torch.randn_like(out)
cg = torch.empty((pb.natoms, 3), device="cuda")
rng = np.random.default_rng(0)
lib = _native.lib()
st = stream_handle(pb.device)
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
n = 100
evs = [[E() for _ in range(5)] for _ in range(n)]


def step(ev=None):
    xf = geom.draw_transform_array(pb.default_centers, 2.0, True, rng)
    if ev: ev[0].record()
    if ev: ev[1].record()
    p = gm._prepare(pb, None, xf, D)
    b = pb.gm_batch()
    if ev: ev[2].record()
    lib.gm_forward(ctypes.byref(p), ctypes.byref(b), pb.workspace.data_ptr(), out.data_ptr(), st)
    if ev: ev[3].record()
    lib.gm_backward(ctypes.byref(p), ctypes.byref(b), pb.workspace.data_ptr(), gg.data_ptr(),
                    cg.data_ptr(), None, st)
    if ev: ev[4].record()


for _ in range(5):
    step()
torch.cuda.synchronize()
for k in range(n):
    step(evs[k])
torch.cuda.synchronize()
names = ["h2d", "prepare", "forward", "backward", "gap to next step"]
acc = [0.0] * 5
for k in range(n - 1):
    for j in range(4):
        acc[j] += evs[k][j].elapsed_time(evs[k][j + 1])
    acc[4] += evs[k][4].elapsed_time(evs[k + 1][0])
for nm, a in zip(names, acc):
    print(f"{nm:20s} {a / (n - 1) * 1e3:8.1f} us")
print(f"{'step':20s} {evs[0][0].elapsed_time(evs[n - 1][0]) / (n - 1) * 1e3:8.1f} us")

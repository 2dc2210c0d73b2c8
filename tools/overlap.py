"""Experiment: step k's backward on a second stream, concurrent with step
k+1's prepare + forward (two packed copies of the batch = two workspaces).
Prints sequential vs pipelined time per step (device events)."""
import sys

sys.path.insert(0, "/root/repo")
import numpy as np
import torch

import bench
from paper_1912_04822_b200 import GridMaker, geom

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = bench.CONFIGS[name]
exs, centers = bench.make_batch(cfg, 0, 1)
gm = GridMaker(resolution=cfg["resolution"], dimension=cfg["dimension"], binary=cfg["binary"])
pbs = [gm.pack(exs), gm.pack(exs)]
D = gm.points_per_side()
outs = [torch.empty((pbs[0].nexamples, pbs[0].nchannels, D, D, D), device="cuda") for _ in range(2)]
gg = torch.randn_like(outs[0])
rng = np.random.default_rng(0)
s_f = torch.cuda.current_stream()
s_b = torch.cuda.Stream(priority=int(sys.argv[2]) if len(sys.argv) > 2 else 0)


def draw():
    return geom.draw_transform_array(pbs[0].default_centers, 2.0, True, rng)


def seq(n):
    for k in range(n):
        gm.forward_packed(pbs[0], outs[0], transforms=draw())
        gm.backward_packed(pbs[0], gg, reuse_prepared=True)


bwd_done = [None, None]


def piped(n):
    for k in range(n):
        x = k & 1
        if bwd_done[x] is not None:
            s_f.wait_event(bwd_done[x])
        gm.forward_packed(pbs[x], outs[x], transforms=draw())
        ev = torch.cuda.Event()
        ev.record(s_f)
        s_b.wait_event(ev)
        with torch.cuda.stream(s_b):
            gm.backward_packed(pbs[x], gg, reuse_prepared=True)
            e2 = torch.cuda.Event()
            e2.record(s_b)
        bwd_done[x] = e2
    s_f.wait_stream(s_b)


for label, fn in (("sequential", seq), ("pipelined", piped), ("sequential", seq),
                  ("pipelined", piped)):
    fn(5)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 50
    a.record()
    fn(n)
    b.record()
    torch.cuda.synchronize()
    print(f"{name} {label}: {a.elapsed_time(b) / n * 1e3:7.1f} us/step")

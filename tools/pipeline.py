"""Serial vs pipelined gridding step (forward of batch k+1 on one stream,
backward of batch k on another), device time per step with CUDA events."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import torch
import bench
from paper_1912_04822_b200 import GridMaker, geom

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
exs, centers = bench.make_batch(cfg, 0, 1)
gm = GridMaker(resolution=cfg["resolution"], dimension=cfg["dimension"], binary=cfg["binary"])
pbs = [gm.pack(exs), gm.pack(exs)]
D = gm.points_per_side()
N, C = pbs[0].nexamples, pbs[0].nchannels
outs = [torch.empty((N, C, D, D, D), device="cuda") for _ in range(2)]
gg = torch.randn((N, C, D, D, D), device="cuda")
cgs = [torch.empty((pbs[0].natoms, 3), device="cuda") for _ in range(2)]
rng = np.random.default_rng(0)
draw = lambda: geom.draw_transform_array(pbs[0].default_centers, 2.0, True, rng)  # noqa: E731
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
main = torch.cuda.current_stream()


def serial(k, grad):
    x = k % 2
    gm.forward_packed(pbs[x], outs[x], transforms=draw())
    gm.backward_packed(pbs[x], outs[x] if grad == "grid" else gg, reuse_prepared=True,
                       coord_grad=cgs[x])


fdone = [torch.cuda.Event(), torch.cuda.Event()]
bdone = [torch.cuda.Event(), torch.cuda.Event()]


def pipelined(k, grad):
    x, y = k % 2, (k + 1) % 2
    with torch.cuda.stream(s1):
        s1.wait_event(bdone[x])          # workspace x free (its backward is done)
        gm.forward_packed(pbs[x], outs[x], transforms=draw())
        fdone[x].record(s1)
    with torch.cuda.stream(s2):
        s2.wait_event(fdone[y])          # batch y was gridded in the previous step
        gm.backward_packed(pbs[y], outs[y] if grad == "grid" else gg, reuse_prepared=True,
                           coord_grad=cgs[y])
        bdone[y].record(s2)


for name, fn in (("serial", serial), ("pipelined", pipelined)):
    for grad in ("random", "grid"):
        for k in range(6):
            fn(k, grad)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 60
        main.wait_stream(s1); main.wait_stream(s2)
        a.record(main)
        s1.wait_stream(main); s2.wait_stream(main)
        for k in range(n):
            fn(k, grad)
        main.wait_stream(s1); main.wait_stream(s2)
        b.record(main)
        torch.cuda.synchronize()
        print(f"{name:10s} grad={grad:6s} {a.elapsed_time(b) / n * 1e3:8.1f} us/step")

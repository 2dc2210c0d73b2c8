"""Fresh-batch step (DatasetBatches, device-assembled) with and without
prefetch: device and host time per step, then a cProfile of the host path.
usage: python tools/fresh_step.py c2|c3"""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
from paper_1912_04822_b200 import GridMaker, geom
from paper_1912_04822_b200.dataset import DeviceDataset
from paper_1912_04822_b200.pipeline import DatasetBatches
name = sys.argv[1]
cfg = bench.CONFIGS[name]
exs, _ = bench.make_batch(cfg, 0, 1, n=1000)
gm = GridMaker(resolution=cfg["resolution"], dimension=cfg["dimension"], binary=cfg["binary"])
ds = DeviceDataset(exs)
D = gm.points_per_side()
out = torch.empty((50, 28, D, D, D), device="cuda")
frng = np.random.default_rng(1)
for prefetch in (False, True, False, True):
    it = DatasetBatches(gm, ds, 50, seed=3, prefetch=prefetch)
    def step(with_copy=True):
        ab = next(it)
        xf = geom.draw_transform_array(ab.default_centers, 2.0, True, frng)
        gm.forward_packed(ab, out[:ab.nexamples], transforms=xf)
        cg, _ = gm.backward_packed(ab, out[:ab.nexamples], reuse_prepared=True)
    for _ in range(5): step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter(); a.record()
    for _ in range(40): step()
    t1 = time.perf_counter(); b.record(); torch.cuda.synchronize()
    print(name, "prefetch", prefetch, "device us/step", a.elapsed_time(b) / 40 * 1e3, "host us/step", (t1 - t) / 40 * 1e6)
import cProfile, pstats
it = DatasetBatches(gm, ds, 50, seed=3, prefetch=True)
def step2():
    ab = next(it)
    xf = geom.draw_transform_array(ab.default_centers, 2.0, True, frng)
    gm.forward_packed(ab, out[:ab.nexamples], transforms=xf)
    gm.backward_packed(ab, out[:ab.nexamples], reuse_prepared=True)
for _ in range(5): step2()
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(200): step2()
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)

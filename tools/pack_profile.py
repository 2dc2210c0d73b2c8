"""cProfile of host packing (GridMaker.pack) of the C2 batch on the GPU box."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, "/root/repo")
import torch

import bench
from paper_1912_04822_b200 import GridMaker

cfg = bench.CONFIGS["c2"]
exs, _ = bench.make_batch(cfg, 0, 1)
gm = GridMaker()
sets = [ex.coord_sets for ex in exs]
for _ in range(3):
    gm.pack(sets)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10):
    gm.pack(sets)
torch.cuda.synchronize()
print("pack ms", (time.perf_counter() - t) * 100)
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    gm.pack(sets)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)

"""cProfile of PackedBatch construction for the C2 batch (host packing cost)."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, "/root/repo")
import bench
from paper_1912_04822_b200 import GridMaker

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
exs, _ = bench.make_batch(cfg, 0, 1)
gm = GridMaker()
sets = [ex.coord_sets for ex in exs]
gm.pack(sets)
t = time.perf_counter()
for _ in range(5):
    gm.pack(sets)
print("pack ms", (time.perf_counter() - t) / 5 * 1e3)
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    gm.pack(sets)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)

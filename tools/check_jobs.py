"""Forward with and without the job table must agree bitwise (quick GPU check)."""
import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_1912_04822_b200 import GridMaker, synthetic, packing
exs = synthetic.batch(3, seed=2)
gm = GridMaker()
a = gm.forward_batch(exs)
packing._NO_JOBS = True
b = gm.forward_batch(exs)
d = np.abs(a - b)
print("max diff", d.max(), "n", (d > 1e-6).sum())
idx = np.argwhere(d > 1e-6)
print(idx[:10])
print("channels with diffs", np.unique(idx[:, 1]), "examples", np.unique(idx[:, 0]), "planes", np.unique(idx[:, 2])[:20])

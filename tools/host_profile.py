import cProfile, pstats, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_1912_04822_b200 import GridMaker, geom, synthetic
exs = synthetic.batch(50, seed=2)
gm = GridMaker(); pb = gm.pack(exs)
out = torch.empty((50, 28, 48, 48, 48), device="cuda"); gg = torch.randn_like(out)
cg = torch.empty((pb.natoms, 3), device="cuda"); rng = np.random.default_rng(0); c = pb.default_centers
def loop(n):
    for _ in range(n):
        gm.forward_packed(pb, out, transforms=geom.draw_transform_array(c, 2.0, True, rng))
        gm.backward_packed(pb, gg, reuse_prepared=True, coord_grad=cg)
loop(5); torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable(); loop(100); pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)

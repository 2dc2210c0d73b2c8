"""Small forward + backward for compute-sanitizer (memcheck / racecheck / synccheck)."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_1912_04822_b200 import GridMaker, synthetic

for binary, vector in ((False, False), (True, False), (False, True)):
    exs = synthetic.batch(2, seed=3, n_receptor=120, vector=vector)
    gm = GridMaker(binary=binary)
    grid, xf = gm.forward_batch(exs, random_rotation=True, random_translation=2.0,
                                rng=np.random.default_rng(0), return_transforms=True)
    if not binary:
        gm.backward_batch(exs, grid, transforms=xf)
gm = GridMaker(resolution=0.25, dimension=23.75)
exs = synthetic.batch(1, seed=3, n_receptor=120, vector=True)
grid = gm.forward_batch(exs)
gm.backward_batch(exs, grid)
print("sanitize run ok")

"""Index-backward footprint at 4-B, 32-B, 64-B and 128-B granularity: the
DRAM-read floor of an atom-centric backward over the (N, C, D, D, D) layout.

    python tools/footprint_granularity.py [c2|c5] [examples]

Counts, over the first few examples of the bench batch (untransformed), the
distinct grid_grad words / sectors / lines inside some same-channel atom's
cutoff, scaled to a 50-grid step.  Round 2, C2: 40.8 / 56.5 / 67.2 / 79.6 MB
against 83 MB of DRAM reads measured by ncu."""
import sys

sys.path.insert(0, "/root/repo")
import numpy as np

import bench

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
NEX = int(sys.argv[2]) if len(sys.argv) > 2 else 6
cfg = bench.CONFIGS[name]
exs, _ = bench.make_batch(cfg, 0, 1)
res = cfg["resolution"]
D = int(round(cfg["dimension"] / res)) + 1
rmult = 1.5
counts = {4: 0, 32: 0, 64: 0, 128: 0}
for ex in exs[:NEX]:
    sets = ex.coord_sets
    origin = sets[-1].coords.astype(np.float64).mean(axis=0) - cfg["dimension"] / 2
    seen = {g: set() for g in counts}
    choff = 0
    for cs in sets:
        xyz = cs.coords.astype(np.float64) - origin
        cut = cs.radii.astype(np.float64) * rmult
        for a in range(len(xyz)):
            c = cut[a]
            lo = np.ceil((xyz[a] - c) / res).clip(0, None).astype(int)
            hi = np.floor((xyz[a] + c) / res).clip(None, D - 1).astype(int)
            if (lo > hi).any():
                continue
            I, J, K = (np.arange(lo[q], hi[q] + 1) for q in range(3))
            d2 = ((I * res - xyz[a, 0])[:, None, None] ** 2 +
                  (J * res - xyz[a, 1])[None, :, None] ** 2 +
                  (K * res - xyz[a, 2])[None, None, :] ** 2)
            ii, jj, kk = np.nonzero(d2 < c * c)
            ch = choff + int(cs.type_index[a])
            addr = ((ch * D + I[ii]) * D + J[jj]) * D + K[kk]  # float index in the slab
            for g in counts:
                seen[g].update((addr // (g // 4)).tolist())
        choff += cs.num_types
    for g in counts:
        counts[g] += len(seen[g])
print(f"{name}: D={D}, {NEX} examples")
for g, n in counts.items():
    print(f"{g:4d}-B granularity: {g * n / NEX * 50 / 1e6:7.1f} MB per 50-grid step")

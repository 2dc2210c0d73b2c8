"""NPY + sidecar fixtures written by the live reference (run in the build
container, where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_npy_golden.py

voxmol.grids.write_npy (grids.py:244-271) and voxmol.voxelizer.save_grid
(voxelizer.py:438-465) on small seeded arrays; the test compares our
export.py output byte for byte."""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from voxmol.grids import write_npy  # noqa: E402
from voxmol.voxelizer import save_grid  # noqa: E402

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "npy")
os.makedirs(HERE, exist_ok=True)
rng = np.random.default_rng(42)
cases = {
    "vec_f32": rng.standard_normal(7).astype(np.float32),
    "grid_f32": rng.standard_normal((2, 3, 5, 5, 5)).astype(np.float32),
    "grid_f64": rng.standard_normal((1, 4, 4, 4)),
    "big_header": rng.standard_normal((3, 28, 6, 6, 6)).astype(np.float32),
}
for name, arr in cases.items():
    np.save(os.path.join(HERE, name + "_input.npy"), arr)
    write_npy(os.path.join(HERE, name + "_ref.npy"), arr)
save_grid(os.path.join(HERE, "saved_ref.npy"), cases["grid_f32"],
          origin=np.array([[-11.75, -11.75, -11.75], [1.0, 2.0, 3.0]]), resolution=0.5,
          channel_labels=[f"rec:{i}" for i in range(3)], extra={"note": "fixture"})
print("wrote", sorted(os.listdir(HERE)))

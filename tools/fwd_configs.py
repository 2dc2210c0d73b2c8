"""k_forward / k_backward device time on the bench configs (CUDA events)."""
import ctypes
import sys

sys.path.insert(0, "/root/repo")
import numpy as np
import torch

import bench
from paper_1912_04822_b200 import GridMaker, _native, geom
from paper_1912_04822_b200.voxelizer import stream_handle

lib = _native.lib()
for name in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["c2", "c5"]):
    cfg = bench.CONFIGS[name]
    exs, centers = bench.make_batch(cfg, 0, 1)
    gm = GridMaker(resolution=cfg["resolution"], dimension=cfg["dimension"], binary=cfg["binary"])
    pb = gm.pack(exs)
    D = gm.points_per_side()
    out = torch.empty((pb.nexamples, pb.nchannels, D, D, D), device="cuda")
    xf = geom.draw_transform_array(pb.default_centers, 2.0, True, np.random.default_rng(0))
    p = gm._prepare(pb, None, xf, D)
    pb.ensure_fwd_jobs(p)  # the job table, as forward_packed uses it
    st = stream_handle(pb.device)
    fn = lambda: lib.gm_forward(ctypes.byref(p), ctypes.byref(pb._gm), pb.workspace.data_ptr(),  # noqa: E731
                                out.data_ptr(), st)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 50
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    print(f"{name} gm_forward {a.elapsed_time(b) / n * 1e3:8.1f} us")

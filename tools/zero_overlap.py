"""Experiment: the forward's scatter tiles (GM_LIB built with GM_FWD_EXP_SKIPZERO)
on one stream, a 400 MB zero fill on another -- how well do they overlap?"""
import ctypes
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import torch
import bench
from paper_1912_04822_b200 import GridMaker, _native, geom
from paper_1912_04822_b200.voxelizer import stream_handle

cfg = bench.CONFIGS["c2"]
exs, centers = bench.make_batch(cfg, 0, 1)
gm = GridMaker()
pb = gm.pack(exs)
D = 48
out = torch.empty((pb.nexamples, pb.nchannels, D, D, D), device="cuda")
zbuf = torch.empty(int(400e6 // 4), device="cuda")
xf = geom.draw_transform_array(pb.default_centers, 2.0, True, np.random.default_rng(0))
p = gm._prepare(pb, None, xf, D)
pb.ensure_fwd_jobs(p)
lib = _native.lib()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def fwd():
    lib.gm_forward(ctypes.byref(p), ctypes.byref(pb._gm), pb.workspace.data_ptr(), out.data_ptr(),
                   s1.cuda_stream)


def timed(label, fn, n=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    main = torch.cuda.current_stream()
    a.record(main)
    s1.wait_stream(main); s2.wait_stream(main)
    for _ in range(n):
        fn()
        s1.wait_stream(s2); s2.wait_stream(s1)  # keep steps aligned
    main.wait_stream(s1); main.wait_stream(s2)
    b.record(main)
    torch.cuda.synchronize()
    print(f"{label:40s} {a.elapsed_time(b) / n * 1e3:8.1f} us")


def zfill():
    with torch.cuda.stream(s2):
        zbuf.zero_()


def zcopy():
    with torch.cuda.stream(s2):
        torch.cuda.current_stream()  # noqa
        zbuf[: zbuf.numel() // 2].copy_(zbuf[zbuf.numel() // 2:], non_blocking=True)


zsrc = torch.zeros(int(200e6 // 4), device="cuda")
cudart = ctypes.CDLL("libcudart.so") if False else None


def zce():
    # D2D memcpy from a zero buffer (may run on a copy engine, not the SMs)
    with torch.cuda.stream(s2):
        zbuf[: zsrc.numel()].copy_(zsrc, non_blocking=True)
        zbuf[zsrc.numel(): 2 * zsrc.numel()].copy_(zsrc, non_blocking=True)


timed("forward (scatter tiles) alone", fwd)
timed("D2D copy 400 MB alone", zce)
timed("forward || D2D copy", lambda: (fwd(), zce()))
timed("zero fill 400 MB alone", zfill)
timed("forward || zero fill", lambda: (fwd(), zfill()))

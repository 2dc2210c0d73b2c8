"""Device time of each piece of the C2 step, each looped alone (CUDA events)."""
import ctypes
import sys

sys.path.insert(0, "/root/repo")
import numpy as np
import torch
from paper_1912_04822_b200 import GridMaker, _native, geom, synthetic
from paper_1912_04822_b200.voxelizer import stream_handle

exs = synthetic.batch(50, seed=2)
gm = GridMaker()
pb = gm.pack(exs)
D = gm.points_per_side()
out = torch.empty((50, 28, D, D, D), device="cuda")
gg = torch.randn_like(out)
cg = torch.empty((pb.natoms, 3), device="cuda")
rng = np.random.default_rng(0)
xf = geom.draw_transform_array(pb.default_centers, 2.0, True, rng)
lib = _native.lib()


def timeit(label, fn, n=200):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    print(f"{label:40s} {a.elapsed_time(b) / n * 1e3:8.1f} us")


p = gm._prepare(pb, None, xf, D)
b = pb.gm_batch()
ws, wsb, st = pb.workspace.data_ptr(), pb.workspace_bytes, stream_handle(pb.device)
timeit("set_call_arrays (H2D)", lambda: pb.set_call_arrays(pb.default_centers - 12.0, xf.packed))
timeit("gm_prepare", lambda: lib.gm_prepare(ctypes.byref(p), ctypes.byref(b), ws, wsb, st))
timeit("_prepare (H2D + prepare)", lambda: gm._prepare(pb, None, xf, D))
timeit("gm_forward", lambda: lib.gm_forward(ctypes.byref(p), ctypes.byref(pb._gm), ws,
                                            out.data_ptr(), st))
timeit("gm_backward", lambda: lib.gm_backward(ctypes.byref(p), ctypes.byref(pb._gm), ws,
                                              gg.data_ptr(), cg.data_ptr(), None, st))
timeit("forward_packed", lambda: gm.forward_packed(pb, out, transforms=xf))
timeit("forward_packed+backward_packed", lambda: (
    gm.forward_packed(pb, out, transforms=xf),
    gm.backward_packed(pb, gg, reuse_prepared=True, coord_grad=cg)))
timeit("step with draw", lambda: (
    gm.forward_packed(pb, out, transforms=geom.draw_transform_array(pb.default_centers, 2.0, True, rng)),
    gm.backward_packed(pb, gg, reuse_prepared=True, coord_grad=cg)))
timeit("torch zero_ of the output (write roofline)", lambda: out.zero_())
timeit("torch copy out <- gg (read+write)", lambda: out.copy_(gg))

# forward of one batch overlapped with the backward of another (two streams)
pb2 = gm.pack(exs)
p2 = gm._prepare(pb2, None, xf, D)
out2 = torch.empty_like(out)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()


def overlapped():
    with torch.cuda.stream(s1):
        lib.gm_forward(ctypes.byref(p), ctypes.byref(pb._gm), ws, out.data_ptr(), s1.cuda_stream)
    with torch.cuda.stream(s2):
        lib.gm_backward(ctypes.byref(p2), ctypes.byref(pb2._gm), pb2.workspace.data_ptr(),
                        gg.data_ptr(), cg.data_ptr(), None, s2.cuda_stream)


for _ in range(5):
    overlapped()
torch.cuda.synchronize()
import time
t = time.perf_counter()
for _ in range(200):
    overlapped()
torch.cuda.synchronize()
print(f"{'fwd || bwd on two streams':40s} {(time.perf_counter() - t) / 200 * 1e6:8.1f} us (wall)")
t = time.perf_counter()
for _ in range(200):
    lib.gm_forward(ctypes.byref(p), ctypes.byref(pb._gm), ws, out.data_ptr(), st)
    lib.gm_backward(ctypes.byref(p2), ctypes.byref(pb2._gm), pb2.workspace.data_ptr(),
                    gg.data_ptr(), cg.data_ptr(), None, st)
torch.cuda.synchronize()
print(f"{'fwd ; bwd on one stream':40s} {(time.perf_counter() - t) / 200 * 1e6:8.1f} us (wall)")

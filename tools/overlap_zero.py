"""Experiment: how much of the forward's zero-slab stores can hide under the
backward.  Splits the forward job table into scatter (work) jobs and zero
jobs and times, per C2 step (device events): each part alone, the backward
alone, zero jobs on a second stream concurrent with the backward, and the
pipelined step [prepare + work jobs (k+1)] -> [backward (k) || zero jobs (k+1)]."""
import ctypes
import sys

sys.path.insert(0, "/root/repo")
import numpy as np
import torch

import bench
from paper_1912_04822_b200 import GridMaker, _native, geom
from paper_1912_04822_b200.packing import stream_handle

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = bench.CONFIGS[name]
exs, centers = bench.make_batch(cfg, 0, 1)
gm = GridMaker(resolution=cfg["resolution"], dimension=cfg["dimension"], binary=cfg["binary"])
D = gm.points_per_side()
pbs = [gm.pack(exs), gm.pack(exs)]
N, C = pbs[0].nexamples, pbs[0].nchannels
outs = [torch.empty((N, C, D, D, D), device="cuda") for _ in range(2)]
gg = torch.randn_like(outs[0])
rng = np.random.default_rng(0)
L = _native.lib()
p = gm._gm_params(D)
parts = []
for pb in pbs:
    xf = geom.draw_transform_array(pb.default_centers, 2.0, True, rng)
    gm._prepare(pb, None, xf, D)
    pb.ensure_fwd_jobs(p)
    jobs = pb._jobs.cpu().numpy()
    off = pb.offsets["chan_off"][0]
    co = pb.host.numpy()[off:off + 4 * N * (C + 1)].view(np.int32).reshape(N, C + 1)
    cnt = jobs[:, 2] - jobs[:, 1]  # job: example | channel << 16, item range, plane | row << 16
    work = torch.from_numpy(np.ascontiguousarray(jobs[cnt > 0])).cuda()
    zero = torch.from_numpy(np.ascontiguousarray(jobs[cnt == 0])).cuda()
    parts.append({"all": (pb._jobs, pb._jobs.shape[0]), "work": (work, work.shape[0]),
                  "zero": (zero, zero.shape[0])})
print({k: v[1] for k, v in parts[0].items()})
s_a = torch.cuda.current_stream()
s_b = torch.cuda.Stream()


def fwd(x, part, stream=None):
    pb = pbs[x]
    t, n = parts[x][part]
    pb._gm.fwd_jobs = t.data_ptr()
    pb._gm.nfwd_jobs = n
    s = stream or s_a
    _native.check(L.gm_forward(ctypes.byref(p), ctypes.byref(pb._gm), pb.workspace.data_ptr(),
                               outs[x].data_ptr(), s.cuda_stream))


def prep(x):
    gm._prepare(pbs[x], None, geom.draw_transform_array(pbs[x].default_centers, 2.0, True, rng), D)


def bwd(x, stream=None):
    with torch.cuda.stream(stream or s_a):
        gm.backward_packed(pbs[x], gg, reuse_prepared=True)


def timeit(label, fn, n=40):
    fn(0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(n):
        fn(k)
    s_a.wait_stream(s_b)
    b.record()
    torch.cuda.synchronize()
    print(f"{name} {label:44s}: {a.elapsed_time(b) / n * 1e3:7.1f} us")


timeit("prepare", lambda k: prep(0))
timeit("forward all (after prepare)", lambda k: fwd(0, "all"))
timeit("forward work jobs", lambda k: fwd(0, "work"))
timeit("forward zero jobs", lambda k: fwd(0, "zero"))
timeit("backward", lambda k: bwd(0))
timeit("step: prep + fwd all + bwd", lambda k: (prep(0), fwd(0, "all"), bwd(0)))


def conc(k):
    ev = torch.cuda.Event()
    ev.record(s_a)
    s_b.wait_event(ev)
    fwd(1, "zero", s_b)
    bwd(0)
    s_a.wait_stream(s_b)


timeit("zero jobs (stream b) || backward", conc)


def fill_conc(k):
    ev = torch.cuda.Event()
    ev.record(s_a)
    s_b.wait_event(ev)
    with torch.cuda.stream(s_b):
        outs[1][:, 10:].fill_(0.0)
    bwd(0)
    s_a.wait_stream(s_b)


timeit("torch fill 18/28 ch (stream b) || backward", fill_conc)


def piped(k):
    x = k & 1
    prep(x)
    fwd(x, "work")
    ev = torch.cuda.Event()
    ev.record(s_a)
    s_b.wait_event(ev)
    fwd(x, "zero", s_b)           # batch k+1's zero slabs ...
    bwd(1 - x)                     # ... under batch k's backward
    s_a.wait_stream(s_b)


timeit("pipelined: prep+work(k+1); bwd(k) || zero(k+1)", piped)

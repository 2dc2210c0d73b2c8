"""Grid-sized host <-> device copies for the numpy-facing API.

The reference returns its grids as numpy arrays (voxelizer.py:223-258) and
takes numpy ``grid_grad``s (voxelizer.py:260-301).  A C2 batch is 620 MB: a
plain ``tensor.cpu()`` into fresh pageable memory measured 293 ms on the box
(page faults plus the driver's pageable staging), an H2D from a pageable
array 57 ms, against 11 ms for one pinned copy (tools/numpy_path.py).

Both directions here stream through two reused pinned chunk buffers: the DMA
of chunk k+1 runs on a side stream while host threads move chunk k between
the pinned buffer and the numpy array (several threads, so the page faults of
a fresh result array are taken in parallel).
"""

from __future__ import annotations

import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

_CHUNK_BYTES = 32 << 20
_LOCK = threading.Lock()
_STAGING = {}  # device index -> _Staging
_POOL = [None, 0]  # executor, its worker count


def _threads() -> int:
    from .voxelizer import get_num_threads

    return max(1, min(16, get_num_threads()))


def _pool() -> ThreadPoolExecutor:
    n = _threads()
    if _POOL[0] is None or _POOL[1] != n:
        if _POOL[0] is not None:
            _POOL[0].shutdown(wait=False)
        _POOL[0] = ThreadPoolExecutor(max_workers=n, thread_name_prefix="gm-hostio")
        _POOL[1] = n
    return _POOL[0]


class _Staging:
    def __init__(self, device):
        self.device = device
        self.bufs = [torch.empty(_CHUNK_BYTES, dtype=torch.uint8, pin_memory=True)
                     for _ in range(2)]
        self.side = torch.cuda.Stream(device=device)
        self.lock = threading.Lock()


def _staging(device) -> _Staging:
    idx = torch.device(device).index
    if idx is None:
        idx = torch.cuda.current_device()
    with _LOCK:
        st = _STAGING.get(idx)
        if st is None:
            st = _STAGING[idx] = _Staging(torch.device("cuda", idx))
    return st


def _parallel_copy(dst: np.ndarray, src: np.ndarray) -> None:
    """dst[:] = src (1-D, same length) split over the host threads."""
    n = dst.shape[0]
    k = _threads()
    if k == 1 or n * dst.itemsize < (4 << 20):
        np.copyto(dst, src)
        return
    step = -(-n // k)
    futs = [_pool().submit(np.copyto, dst[s:s + step], src[s:s + step])
            for s in range(0, n, step)]
    for f in futs:
        f.result()


def to_host(t: torch.Tensor, out: np.ndarray | None = None) -> np.ndarray:
    """Copy a CUDA tensor into ``out`` (or a new array of its shape/dtype)."""
    t = t.detach()
    if not t.is_contiguous():
        t = t.contiguous()
    np_dtype = torch.empty(0, dtype=t.dtype).numpy().dtype
    if out is None:
        out = np.empty(tuple(t.shape), dtype=np_dtype)
    flat_out = out.reshape(-1)
    if flat_out.dtype != np_dtype or flat_out.size != t.numel() or not out.flags.c_contiguous:
        raise ValueError("out must be a C-contiguous array of the tensor's size and dtype")
    src = t.view(-1).view(torch.uint8)
    dst = flat_out.view(np.uint8)
    nbytes = src.numel()
    if nbytes == 0:
        return out
    st = _staging(t.device)
    with st.lock:
        st.side.wait_stream(torch.cuda.current_stream(t.device))  # the producer of `t`
        starts = list(range(0, nbytes, _CHUNK_BYTES))
        events = [None, None]

        def issue(k):
            s = starts[k]
            m = min(_CHUNK_BYTES, nbytes - s)
            with torch.cuda.stream(st.side):
                st.bufs[k % 2][:m].copy_(src[s:s + m], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(st.side)
            events[k % 2] = ev

        issue(0)
        for k, s in enumerate(starts):
            if k + 1 < len(starts):
                issue(k + 1)  # its buffer's last host copy (chunk k-1) is done
            events[k % 2].synchronize()
            m = min(_CHUNK_BYTES, nbytes - s)
            _parallel_copy(dst[s:s + m], st.bufs[k % 2].numpy()[:m])
        t.record_stream(st.side)
    return out


def to_device(a: np.ndarray, device, dtype=np.float32) -> torch.Tensor:
    """A CUDA tensor copy of numpy array ``a`` (converted to ``dtype``),
    ordered before later work on the current stream."""
    a = np.ascontiguousarray(a, dtype=dtype)
    dev = torch.device(device)
    out = torch.empty(a.shape, dtype=torch.from_numpy(a[:0].reshape(-1)).dtype, device=dev)
    src = a.reshape(-1).view(np.uint8)
    nbytes = src.shape[0]
    if nbytes == 0:
        return out
    dst = out.view(-1).view(torch.uint8)
    st = _staging(dev)
    cur = torch.cuda.current_stream(dev)
    with st.lock:
        st.side.wait_stream(cur)  # `out` was allocated on the current stream
        events = [None, None]
        for k, s in enumerate(range(0, nbytes, _CHUNK_BYTES)):
            m = min(_CHUNK_BYTES, nbytes - s)
            if events[k % 2] is not None:
                events[k % 2].synchronize()  # this buffer's previous DMA is done
            _parallel_copy(st.bufs[k % 2].numpy()[:m], src[s:s + m])
            with torch.cuda.stream(st.side):
                dst[s:s + m].copy_(st.bufs[k % 2][:m], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(st.side)
            events[k % 2] = ev
        cur.wait_stream(st.side)
        out.record_stream(st.side)
        # the pinned buffers are reused by the next call: wait for the last DMAs
        for ev in events:
            if ev is not None:
                ev.synchronize()
    return out

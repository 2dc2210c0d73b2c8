"""Grid-sized host <-> device copies for the numpy-facing API.

The reference returns its grids as numpy arrays (voxelizer.py:223-258) and
takes numpy ``grid_grad``s (voxelizer.py:260-301).  A C2 batch is 620 MB: a
plain ``tensor.cpu()`` into fresh pageable memory measured 293 ms on the box
(page faults plus the driver's pageable staging), an H2D from a pageable
array 57 ms, against 11 ms for one pinned copy (tools/numpy_path.py).

Results go straight into pinned blocks lent from a small pool (``pinned_result``):
one DMA at full PCIe speed, no fresh pages; a block returns to the pool when
the last numpy array viewing it dies (the arrays reference the block's owner
through their ctypes base, so views keep it too).  Otherwise both directions stream through two
reused pinned chunk buffers: the DMA of chunk k+1 runs on a side stream while
host threads move chunk k between the pinned buffer and the numpy array
(several threads, so the page faults of a fresh result array are taken in
parallel).
"""

from __future__ import annotations

import ctypes
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

_CHUNK_BYTES = 32 << 20
_LOCK = threading.Lock()
_STAGING = {}  # device index -> _Staging
_POOL = [None, 0]  # executor, its worker count
# lent pinned result blocks: at most _RESULT_BLOCKS per size, _RESULT_CAP bytes
_RESULT_BLOCKS = 2
_RESULT_CAP = 4 << 30
_RESULTS = {"free": {}, "count": {}, "bytes": 0, "ranges": {}}


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
    if is_pooled(a):  # already pinned: one DMA
        return torch.from_numpy(a).to(dev)
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


def _release(storage, nbytes):
    with _LOCK:
        _RESULTS["free"].setdefault(nbytes, []).append(storage)


class _Lent:
    """Owner of a lent block: referenced (through a ctypes array) by the numpy
    array built on the block and by all of its views; the block returns to the
    pool when the last of them is gone."""

    def __init__(self, storage, nbytes):
        self.storage, self.nbytes = storage, nbytes

    def __del__(self):
        try:
            _release(self.storage, self.nbytes)
        except Exception:  # interpreter shutdown: the pool is gone anyway
            pass


def pinned_result(shape, dtype=np.float32):
    """A numpy array on a pinned block lent from the result pool, or None when
    the pool is at its limits."""
    dtype = np.dtype(dtype)
    n = 1
    for d in shape:
        n *= int(d)
    nbytes = n * dtype.itemsize
    if nbytes == 0:
        return None
    with _LOCK:
        free = _RESULTS["free"].get(nbytes)
        storage = free.pop() if free else None
        if storage is None:
            if _RESULTS["count"].get(nbytes, 0) >= _RESULT_BLOCKS or \
                    _RESULTS["bytes"] + nbytes > _RESULT_CAP:
                return None
            _RESULTS["count"][nbytes] = _RESULTS["count"].get(nbytes, 0) + 1
            _RESULTS["bytes"] += nbytes
    if storage is None:
        storage = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True).untyped_storage()
        with _LOCK:
            _RESULTS["ranges"][storage.data_ptr()] = nbytes
    raw = (ctypes.c_char * nbytes).from_address(storage.data_ptr())
    raw._lent = _Lent(storage, nbytes)
    return np.frombuffer(raw, dtype=dtype, count=n).reshape(tuple(shape))


def is_pooled(a: np.ndarray) -> bool:
    """Whether numpy array ``a`` lies inside a pinned block of the result pool."""
    try:
        p = a.__array_interface__["data"][0]
    except (AttributeError, KeyError, TypeError):
        return False
    with _LOCK:
        for base, nb in _RESULTS["ranges"].items():
            if base <= p and p + a.nbytes <= base + nb:
                return True
    return False


def grid_to_numpy(t: torch.Tensor) -> np.ndarray:
    """A fresh numpy array holding CUDA tensor ``t``: one pinned DMA into a
    pooled block when one is free, else ``to_host``."""
    t = t.detach()
    host = pinned_result(tuple(t.shape), torch.empty(0, dtype=t.dtype).numpy().dtype)
    if host is None:
        return to_host(t)
    torch.from_numpy(host).copy_(t)  # pinned destination: one DMA
    return host

"""Grid export: NPY v1.0 + JSON sidecar.

Byte-compatible with the reference's writer
(/root/reference/pkg/src/voxmol/grids.py:244-271 ``write_npy``,
voxelizer.py:438-465 ``save_grid``): the same header dictionary, padded with
spaces so magic + version + length + header is a multiple of 64 bytes, then
the little-endian C-order payload.

Device grids (a C2 batch is 620 MB) stream device -> pinned -> file in
chunks: two pinned buffers alternate, the copy of chunk k+1 runs on a side
stream while chunk k is written, so the host never holds the whole batch.
"""

from __future__ import annotations

import ast
import json
import os
import struct

import numpy as np

from . import errors

_NPY_MAGIC = b"\x93NUMPY"


def _descr_of(dtype) -> str:
    dt = np.dtype(dtype)
    if dt == np.float32:
        return "<f4"
    if dt == np.float64:
        return "<f8"
    raise TypeError(f"only float32/float64 grids serialize to NPY, got {dt}")


def npy_header(shape, descr: str) -> bytes:
    """magic + version 1.0 + header length + padded header (grids.py:253-264)."""
    shape = tuple(int(d) for d in shape)
    shape_repr = repr(shape) if len(shape) != 1 else f"({shape[0]},)"
    header = f"{{'descr': '{descr}', 'fortran_order': False, 'shape': {shape_repr}, }}"
    unpadded = len(_NPY_MAGIC) + 2 + 2 + len(header) + 1
    header = header + " " * ((64 - unpadded % 64) % 64) + "\n"
    return _NPY_MAGIC + bytes([1, 0]) + struct.pack("<H", len(header)) + header.encode("latin1")


def _torch():
    try:
        import torch
    except ImportError:  # pragma: no cover
        return None
    return torch


def _is_cuda_tensor(x) -> bool:
    torch = _torch()
    return torch is not None and isinstance(x, torch.Tensor) and x.is_cuda


def write_npy(path, array, chunk_bytes: int = 64 << 20) -> None:
    """Write a numpy array, grid view (``.array``) or tensor as NPY v1.0.

    CUDA tensors stream through two pinned chunk buffers (no full host copy).
    """
    torch = _torch()
    if not isinstance(array, np.ndarray) and not (torch is not None and isinstance(array, torch.Tensor)) \
            and hasattr(array, "array"):
        array = array.array  # grid views (grids.py:161-225)
    if _is_cuda_tensor(array):
        _write_npy_device(path, array, chunk_bytes)
        return
    if torch is not None and isinstance(array, torch.Tensor):
        array = array.detach().numpy()
    array = np.ascontiguousarray(array)
    descr = _descr_of(array.dtype)
    with open(path, "wb") as fh:
        fh.write(npy_header(array.shape, descr))
        fh.write(array.astype(descr, copy=False).tobytes())


def _write_npy_device(path, t, chunk_bytes: int) -> None:
    torch = _torch()
    t = t.detach()
    if t.dtype not in (torch.float32, torch.float64):
        raise TypeError(f"only float32/float64 grids serialize to NPY, got {t.dtype}")
    t = t.contiguous()
    descr = "<f4" if t.dtype == torch.float32 else "<f8"
    flat = t.view(-1)
    esz = flat.element_size()
    per = max(1, int(chunk_bytes) // esz)
    bufs = [torch.empty(min(per, max(flat.numel(), 1)), dtype=t.dtype, pin_memory=True)
            for _ in range(2)]
    side = torch.cuda.Stream(device=t.device)
    side.wait_stream(torch.cuda.current_stream(t.device))  # the producer of `t`
    events = [None, None]
    with open(path, "wb") as fh:
        fh.write(npy_header(tuple(t.shape), descr))
        n = flat.numel()
        starts = list(range(0, n, per))

        def issue(k):
            s = starts[k]
            m = min(per, n - s)
            slot = k % 2
            with torch.cuda.stream(side):
                bufs[slot][:m].copy_(flat[s:s + m], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(side)
            events[slot] = ev
            return m

        sizes = {}
        if starts:
            sizes[0] = issue(0)
        for k in range(len(starts)):
            if k + 1 < len(starts):
                # the buffer of chunk k+1 was last written to the file at k-1
                sizes[k + 1] = issue(k + 1)
            events[k % 2].synchronize()
            fh.write(bufs[k % 2][:sizes[k]].numpy().tobytes())
    # keep `t` alive until the side stream is done with it
    t.record_stream(side)


def read_npy(path) -> np.ndarray:
    """Read an NPY v1.0 file (grids.py:274-307 semantics and errors)."""
    with open(path, "rb") as fh:
        magic = fh.read(6)
        if magic != _NPY_MAGIC:
            raise errors.FormatError(f"{path}: not an NPY file (bad magic {magic!r})")
        version = fh.read(2)
        if len(version) < 2 or version[0] != 1:
            raise errors.FormatError(f"{path}: unsupported NPY version {tuple(version)!r}")
        raw_len = fh.read(2)
        if len(raw_len) < 2:
            raise errors.FormatError(f"{path}: truncated NPY header")
        (hlen,) = struct.unpack("<H", raw_len)
        header = fh.read(hlen)
        if len(header) < hlen:
            raise errors.FormatError(f"{path}: truncated NPY header")
        try:
            meta = ast.literal_eval(header.decode("latin1"))
        except (ValueError, SyntaxError) as exc:
            raise errors.FormatError(f"{path}: unparseable NPY header") from exc
        descr = meta.get("descr")
        if descr not in ("<f4", "<f8"):
            raise errors.FormatError(f"{path}: unsupported descr {descr!r}, expected <f4/<f8")
        if meta.get("fortran_order"):
            raise errors.FormatError(f"{path}: fortran-order NPY files are not supported")
        shape = tuple(meta.get("shape", ()))
        count = int(np.prod(shape)) if shape else 1
        payload = fh.read()
    expected = count * np.dtype(descr).itemsize
    if len(payload) < expected:
        raise errors.FormatError(f"{path}: truncated NPY payload ({len(payload)} < {expected} bytes)")
    return np.frombuffer(payload[:expected], dtype=descr).reshape(shape).copy()


def save_grid(path, grid, origin=None, resolution=None, channel_labels=None,
              extra=None) -> str:
    """NPY + JSON sidecar (voxelizer.py:438-465); returns the sidecar path.

    ``grid`` may be a numpy array, a grid view or a (CUDA) tensor."""
    path = os.fspath(path)
    write_npy(path, grid)
    arr = grid.array if (hasattr(grid, "array") and not hasattr(grid, "dtype")) else grid
    shape = tuple(arr.shape) if hasattr(arr, "shape") else tuple(np.asarray(arr).shape)
    meta = {"shape": [int(d) for d in shape]}
    if resolution is not None:
        meta["resolution"] = float(resolution)
    if origin is not None:
        o = np.asarray(origin, dtype=np.float64)
        if o.ndim == 1:
            meta["origin"] = [float(v) for v in o]
        else:
            meta["origins"] = [[float(v) for v in row] for row in o]
    if channel_labels is not None:
        meta["channels"] = list(channel_labels)
    if extra:
        meta.update(extra)
    sidecar = os.path.splitext(path)[0] + ".json"
    with open(sidecar, "w", encoding="utf-8") as fh:
        json.dump(meta, fh, indent=2, sort_keys=True)
        fh.write("\n")
    return sidecar

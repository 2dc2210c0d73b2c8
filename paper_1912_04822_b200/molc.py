"""MOLC structure cache -> typed atoms, host or device.

The reference reads its binary cache (/root/reference/pkg/src/voxmol/
chemio.py:227-391) into one ``RawAtom`` Python object per atom
(chemio.py:353-356) and types them one by one (atomtypes.py:272-291).  Here
a cache is memory-mapped once and every entry is a zero-copy numpy view of
its 13-byte records; typing is a table lookup over the element column.

* ``MolcCache.typed(name)``: the ``CoordinateSet`` the reference's
  ``type_molecule(cache.lookup(name), default_element_typer())`` builds,
  bit for bit (same f32 coordinates, atom order, radii, types).
* ``MolcCache.to_device(names)``: the raw records of many entries copied
  (one slice per entry) into one pinned buffer, one host->device copy, then
  decoded and typed on the device by ``gm_molc_decode`` (csrc/molc.cu):
  (natoms, 3) f32 coordinates, type index, radius and per-entry offsets -- no
  per-atom host work at all.

Layout (little-endian): "MOLC", u32 version 1, u64 count, entries (u16 name
length, UTF-8 name, u32 natoms, natoms x (u8 element, 3 x f32)), index
sorted by name (u16 length, name, u64 entry offset), u64 index offset.
"""

from __future__ import annotations

import mmap
import os
import struct

import numpy as np

from .coordsets import CoordinateSet
from . import errors

MOLC_MAGIC = b"MOLC"
MOLC_VERSION = 1
ATOM_DTYPE = np.dtype([("element", "u1"), ("x", "<f4"), ("y", "<f4"), ("z", "<f4")])
assert ATOM_DTYPE.itemsize == 13


# ---------------------------------------------------------------------------
# element typing table (atomtypes.py:191-228, the default 14-type table)
# ---------------------------------------------------------------------------
TYPE_NAMES = ["C", "N", "O", "S", "P", "F", "Cl", "Br", "I", "B", "Si", "Se", "Metal", "Other"]
TYPE_RADII = np.array([1.90, 1.80, 1.70, 2.00, 2.10, 1.50, 1.80, 2.00, 2.20, 1.92, 2.20, 1.90,
                       1.20, 1.70], dtype=np.float32)
_SINGLE = {"C": 6, "N": 7, "O": 8, "S": 16, "P": 15, "F": 9, "Cl": 17, "Br": 35, "I": 53,
           "B": 5, "Si": 14, "Se": 34}
_METALS = ((3, 4, 11, 12, 13) + tuple(range(19, 32)) + tuple(range(37, 51))
           + tuple(range(55, 84)) + (87, 88) + tuple(range(89, 104)))
_OTHER = (32, 33, 51, 52, 84, 85)


def element_type_table() -> np.ndarray:
    """(256,) int16: element number -> type index, -1 = atom dropped
    (hydrogens, noble gases and unmapped elements, atomtypes.py:125-135)."""
    t = np.full(256, -1, np.int16)
    for sym, z in _SINGLE.items():
        t[z] = TYPE_NAMES.index(sym)
    for z in _METALS:
        if t[z] < 0:
            t[z] = TYPE_NAMES.index("Metal")
    for z in _OTHER:
        t[z] = TYPE_NAMES.index("Other")
    return t


class MolcCache:
    """Read side of a MOLC cache: memory-mapped, index-directed lookups."""

    def __init__(self, path):
        self.path = os.fspath(path)
        self._fh = open(self.path, "rb")
        try:
            if os.fstat(self._fh.fileno()).st_size < 24:
                raise errors.FormatError(f"{self.path}: file too small to be a MOLC cache")
            self._mm = mmap.mmap(self._fh.fileno(), 0, access=mmap.ACCESS_READ)
            self._buf = np.frombuffer(self._mm, dtype=np.uint8)
            self._index = self._load_index()
        except Exception:
            self.close()
            raise
        self._types = element_type_table()

    def _load_index(self) -> dict:
        mm = self._mm
        if mm[:4] != MOLC_MAGIC:
            raise errors.FormatError(f"{self.path}: bad magic {bytes(mm[:4])!r}")
        (version,) = struct.unpack_from("<I", mm, 4)
        if version != MOLC_VERSION:
            raise errors.FormatError(f"{self.path}: unsupported cache version {version}")
        (count,) = struct.unpack_from("<Q", mm, 8)
        (index_offset,) = struct.unpack_from("<Q", mm, len(mm) - 8)
        if not 16 <= index_offset <= len(mm) - 8:
            raise errors.FormatError(f"{self.path}: index offset {index_offset} out of range")
        index, pos = {}, index_offset
        try:
            for _ in range(count):
                (nlen,) = struct.unpack_from("<H", mm, pos)
                name = bytes(mm[pos + 2:pos + 2 + nlen]).decode("utf-8")
                (off,) = struct.unpack_from("<Q", mm, pos + 2 + nlen)
                pos += 10 + nlen
                if not 16 <= off < index_offset:
                    raise errors.FormatError(f"{self.path}: entry offset {off} out of range")
                index[name] = off
        except (struct.error, UnicodeDecodeError) as exc:
            raise errors.FormatError(f"{self.path}: truncated or corrupt index") from exc
        if pos != len(mm) - 8:
            raise errors.FormatError(f"{self.path}: index does not span to footer")
        return index

    # -- lookups -----------------------------------------------------------
    def _span(self, name: str) -> tuple[int, int]:
        """(byte offset of the first record, natoms) of one entry."""
        if self._mm is None:
            raise RuntimeError(f"cache {self.path} is closed")
        try:
            off = self._index[name]
        except KeyError:
            raise KeyError(f"structure {name!r} not found in {self.path}") from None
        try:
            (nlen,) = struct.unpack_from("<H", self._mm, off)
            off += 2 + nlen
            (natoms,) = struct.unpack_from("<I", self._mm, off)
        except struct.error as exc:
            raise errors.FormatError(f"{self.path}: truncated entry for {name!r}") from exc
        off += 4
        if off + natoms * ATOM_DTYPE.itemsize > len(self._mm):
            raise errors.FormatError(f"{self.path}: truncated entry for {name!r}")
        return off, natoms

    def records(self, name: str) -> np.ndarray:
        """Zero-copy structured view (element, x, y, z) of one entry."""
        off, n = self._span(name)
        return self._buf[off:off + n * ATOM_DTYPE.itemsize].view(ATOM_DTYPE)

    def typed(self, name: str) -> CoordinateSet:
        """atomtypes.type_molecule(lookup(name), default_element_typer())."""
        rec = self.records(name)
        t = self._types[rec["element"]]
        keep = t >= 0
        r = rec[keep]
        coords = np.empty((r.shape[0], 3), np.float32)
        coords[:, 0], coords[:, 1], coords[:, 2] = r["x"], r["y"], r["z"]
        ti = t[keep].astype(np.int64)
        return CoordinateSet(coords=coords, radii=TYPE_RADII[ti], num_types=len(TYPE_NAMES),
                             type_index=ti, type_names=list(TYPE_NAMES),
                             type_radii=TYPE_RADII.copy())

    def to_device(self, names, device="cuda"):
        """Raw records of ``names`` -> one pinned buffer -> one H2D copy ->
        decode + typing on the device (``gm_molc_decode``: three sm_100a
        kernels, in-order compaction of the kept atoms).  Returns a dict of
        CUDA tensors: ``coords`` (A, 3) f32, ``type_index`` (A,) int32,
        ``radius`` (A,) f32 and ``offsets`` (len(names)+1,) int64 (entry e owns
        atoms [offsets[e], offsets[e+1]) after dropping untyped atoms)."""
        import torch

        from . import _native
        from .packing import on_device, stream_handle

        dev = torch.device(device)
        spans = [self._span(n) for n in names]
        counts = np.array([n for _, n in spans], np.int64)
        total = int(counts.sum())
        starts = np.zeros(len(names) + 1, np.int64)
        np.cumsum(counts, out=starts[1:])
        hdr = starts.nbytes
        pinned = torch.empty(hdr + max(total, 1) * ATOM_DTYPE.itemsize, dtype=torch.uint8,
                             pin_memory=True)
        host = pinned.numpy()
        host[:hdr] = starts.view(np.uint8)
        pos = hdr
        for off, n in spans:  # one slice copy per entry
            nb = n * ATOM_DTYPE.itemsize
            host[pos:pos + nb] = self._buf[off:off + nb]
            pos += nb
        buf = pinned.to(dev, non_blocking=True)
        table, radii = self._device_tables(dev)
        coords = torch.empty((max(total, 1), 3), dtype=torch.float32, device=dev)
        type_index = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
        radius = torch.empty(max(total, 1), dtype=torch.float32, device=dev)
        offsets = torch.empty(len(names) + 1, dtype=torch.int64, device=dev)
        with on_device(dev):
            _native.check(_native.lib().gm_molc_decode(
                buf.data_ptr() + hdr, buf.data_ptr(), len(names), table.data_ptr(),
                radii.data_ptr(), coords.data_ptr(), type_index.data_ptr(), radius.data_ptr(),
                offsets.data_ptr(), stream_handle(dev)))
        kept = int(offsets[-1].item())  # the outputs' length (one 8-byte read back)
        return {"coords": coords[:kept], "type_index": type_index[:kept],
                "radius": radius[:kept], "offsets": offsets}

    def _device_tables(self, dev):
        """The element -> type table (int16) and the type radii on ``dev``,
        uploaded once per device."""
        import torch

        cache = self.__dict__.setdefault("_dev_tables", {})
        key = str(dev)
        if key not in cache:
            cache[key] = (torch.from_numpy(self._types.astype(np.int16)).to(dev),
                          torch.from_numpy(TYPE_RADII).to(dev))
        return cache[key]

    def names(self) -> list:
        return sorted(self._index)

    def __contains__(self, name) -> bool:
        return name in self._index

    def __len__(self) -> int:
        return len(self._index)

    def close(self) -> None:
        self._buf = None
        if getattr(self, "_mm", None) is not None:
            try:
                self._mm.close()
            except BufferError:  # record views still alive: unmapped when they die
                pass
            self._mm = None
        if getattr(self, "_fh", None) is not None:
            self._fh.close()
            self._fh = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def write_molc(molecules, path) -> None:
    """Write (name, elements (n,) u8, coords (n,3) f32) tuples as a MOLC cache
    (chemio.py:242-276 layout; duplicate names: the last one wins)."""
    unique = {}
    for name, elements, coords in molecules:
        unique[name] = (np.asarray(elements, np.uint8), np.asarray(coords, np.float32))
    offsets = {}
    with open(path, "wb") as fh:
        fh.write(MOLC_MAGIC + struct.pack("<I", MOLC_VERSION) + struct.pack("<Q", len(unique)))
        for name, (el, xyz) in unique.items():
            nb = name.encode("utf-8")
            if len(nb) > 0xFFFF:
                raise ValueError(f"structure name too long ({len(nb)} bytes)")
            offsets[name] = fh.tell()
            rec = np.empty(el.shape[0], ATOM_DTYPE)
            rec["element"], rec["x"], rec["y"], rec["z"] = el, xyz[:, 0], xyz[:, 1], xyz[:, 2]
            fh.write(struct.pack("<H", len(nb)) + nb + struct.pack("<I", el.shape[0]))
            fh.write(rec.tobytes())
        index_offset = fh.tell()
        for name in sorted(offsets):
            nb = name.encode("utf-8")
            fh.write(struct.pack("<H", len(nb)) + nb + struct.pack("<Q", offsets[name]))
        fh.write(struct.pack("<Q", index_offset))

"""Host-side packing of examples into one device-resident CSR batch.

Restates the packing of the reference's ``GridMaker._run_batch``
(/root/reference/pkg/src/voxmol/voxelizer.py:372-435) for the C ABI's
``gm_batch``: atoms of every set of every example are concatenated in
example/set order; sets own consecutive channel blocks (``set_choff``);
radii are widened to f64 and multiplied by ``radius_scale`` on the host
exactly like voxelizer.py:416,430; vector-mode forward items are the
nonzero weights in atom-major, channel-minor order (_kernels.py:159-166).

All static arrays live in ONE pinned host buffer mirrored by ONE device
buffer, so (re)uploading a batch is a single host->device copy.  The
per-call arrays (origins, transforms) are uploaded separately.
"""

from __future__ import annotations

import contextlib
import ctypes
import os

import numpy as np
import torch

from . import _native
from . import errors

_ALIGN = 256
# GM_NO_JOBS=1: dense forward launch (A/B timing of the job table)
_NO_JOBS = os.environ.get("GM_NO_JOBS", "") not in ("", "0")
# GM_PACK=numpy: index-typed batches packed by the numpy code below instead of
# the native packer (gm_pack_index_host); the two are compared in the tests
_NATIVE_PACK = os.environ.get("GM_PACK", "native") != "numpy"


class _Layout:
    def __init__(self):
        self.arrays = []   # (name, np.ndarray)
        self.offsets = {}
        self.size = 0

    def add(self, name, arr):
        arr = np.ascontiguousarray(arr)
        self.offsets[name] = (self.size, arr.dtype, arr.shape)
        self.arrays.append((name, arr))
        self.size += (arr.nbytes + _ALIGN - 1) // _ALIGN * _ALIGN if arr.nbytes else _ALIGN

    def reserve(self, name, dtype, shape):
        """Room for an array another writer fills in place (the native packer)."""
        dtype = np.dtype(dtype)
        nbytes = int(np.prod(shape)) * dtype.itemsize
        self.offsets[name] = (self.size, dtype, tuple(shape))
        self.size += (nbytes + _ALIGN - 1) // _ALIGN * _ALIGN if nbytes else _ALIGN


class PackedBatch:
    """A batch of examples resident in device memory.

    Attributes of interest: ``nexamples``, ``nchannels``, ``natoms``,
    ``placed`` (list of (example, choff, set, atom_offset, weight_offset)),
    ``default_centers`` (N,3) float64 (voxelizer.py:305-309 semantics).
    """

    def __init__(self, example_sets, nchannels, vector_mode, radius_scale,
                 radius_type_indexed, device, centers=None):
        self.device = torch.device(device)
        self.nexamples = len(example_sets)
        self.nchannels = int(nchannels)
        self.vector_mode = bool(vector_mode)
        placed = []
        for e, sets in enumerate(example_sets):
            choff = 0
            for cs in sets:
                placed.append((e, choff, cs))
                choff += int(cs.num_types)
        self.nsets = len(placed)
        counts = np.array([int(cs.coords.shape[0]) for _, _, cs in placed], dtype=np.int64)
        starts = np.zeros(self.nsets, np.int64)
        if self.nsets:
            starts[1:] = np.cumsum(counts)[:-1]
        self.natoms = int(counts.sum())
        scale = float(radius_scale)
        if not self.vector_mode and _NATIVE_PACK and _BWD_ORDER in ("slab", "none"):
            self._pack_index_native(example_sets, placed, counts, starts, scale)
            return
        if self.vector_mode and _NATIVE_PACK and _BWD_ORDER in ("slab", "lpt", "lpt_local", "none"):
            self._pack_vector_native(example_sets, placed, counts, starts, scale,
                                     bool(radius_type_indexed))
            return

        coords = np.zeros((self.natoms, 3), np.float32)
        radius = np.zeros(self.natoms, np.float64)
        atom_set = np.zeros(self.natoms, np.int32)
        set_start = starts.astype(np.int32)
        set_end = (starts + counts).astype(np.int32)
        set_example = np.array([p[0] for p in placed], np.int32)
        set_choff = np.array([p[1] for p in placed], np.int32)
        set_t = np.array([int(p[2].num_types) for p in placed], np.int32)
        for s, (e, choff, cs) in enumerate(placed):
            a0, a1 = starts[s], starts[s] + counts[s]
            if a1 > a0:
                coords[a0:a1] = cs.coords
                radius[a0:a1] = cs.radii.astype(np.float64) * scale
            atom_set[a0:a1] = s

        self.atom_example = set_example[atom_set] if self.natoms else np.zeros(0, np.int32)
        # voxelizer.py:305-309 defaults (also the backward's launch-order proxy)
        self.default_centers = np.stack([_default_center(sets) for sets in example_sets]) \
            if self.nexamples else np.zeros((0, 3))

        L = _Layout()
        L.add("coords32", coords)
        L.add("atom_radius", radius)
        L.add("atom_set", atom_set)
        for name, arr in (("set_start", set_start), ("set_end", set_end),
                          ("set_example", set_example), ("set_choff", set_choff),
                          ("set_t", set_t)):
            L.add(name, arr)

        self.placed = []
        ex_start = np.zeros(self.nexamples, np.int32)
        ex_end = np.zeros(self.nexamples, np.int32)
        if not self.vector_mode:
            atom_type = np.zeros(self.natoms, np.int32)
            for s, (e, choff, cs) in enumerate(placed):
                a0, a1 = starts[s], starts[s] + counts[s]
                if a1 > a0:
                    atom_type[a0:a1] = cs.type_index
                self.placed.append((e, choff, cs, int(a0), -1))
            L.add("atom_type", atom_type)
            slot = _bwd_slots(coords, self.atom_example, self.default_centers,
                              slab=self.atom_example.astype(np.int64) * max(self.nchannels, 1) +
                              set_choff[atom_set] + atom_type if self.natoms else None)
            self._bwd_slot_host = slot
            if slot is not None:
                L.add("bwd_slot", slot)
            for s in range(self.nsets):
                e = set_example[s]
                if s == 0 or set_example[s - 1] != e:
                    ex_start[e] = set_start[s]
                ex_end[e] = set_end[s]
            self.nitems = self.natoms
            self.nweights = 0
        else:
            wparts, trparts, it_atom, it_ch, it_w, it_r, it_wi = [], [], [], [], [], [], []
            set_wstart = np.zeros(self.nsets, np.int32)
            set_trstart = np.zeros(self.nsets, np.int32)
            wpos = tpos = ipos = 0
            for s, (e, choff, cs) in enumerate(placed):
                na, nt = int(counts[s]), int(cs.num_types)
                a0 = int(starts[s])
                if s == 0 or set_example[s - 1] != e:
                    ex_start[e] = ipos
                set_wstart[s] = wpos
                set_trstart[s] = tpos
                tv = (np.zeros((0, nt), np.float32) if cs.type_vector is None
                      else np.asarray(cs.type_vector, np.float32))
                if radius_type_indexed and na:
                    if cs.type_radii is None:
                        raise errors.ConfigError(
                            "radius_type_indexed requires coordinate sets typed from a table "
                            "(type_radii is missing)")
                    tr = cs.type_radii.astype(np.float64) * scale
                else:
                    tr = np.ones(nt, np.float64)
                wparts.append(tv.reshape(-1))
                trparts.append(tr)
                if na:
                    ia, ic = np.nonzero(tv)  # row-major: atom-major, channel-minor
                    it_atom.append((ia + a0).astype(np.int32))
                    it_ch.append(ic.astype(np.int32))
                    it_w.append(tv[ia, ic].astype(np.float32))
                    it_r.append(tr[ic] if radius_type_indexed else radius[ia + a0])
                    it_wi.append((wpos + ia * nt + ic).astype(np.int64))
                    ipos += ia.shape[0]
                ex_end[e] = ipos
                self.placed.append((e, choff, cs, a0, int(wpos)))
                wpos += na * nt
                tpos += nt
            cat = (lambda parts, dt: np.concatenate(parts).astype(dt) if parts
                   else np.zeros(0, dt))
            L.add("weights", cat(wparts, np.float32))
            L.add("type_radius", cat(trparts, np.float64))
            L.add("set_wstart", set_wstart)
            L.add("set_trstart", set_trstart)
            L.add("item_atom", cat(it_atom, np.int32))
            L.add("item_channel", cat(it_ch, np.int32))
            L.add("item_weight", cat(it_w, np.float32))
            L.add("item_radius", cat(it_r, np.float64))
            self.nitems = int(ipos)
            self.nweights = int(wpos)
            slot = _bwd_slots(coords, self.atom_example, self.default_centers,
                              per_example=True)
            if slot is not None:
                L.add("bwd_slot", slot)
            # item -> its entry of the packed weight rows (autograd weight refresh)
            self.item_windex = cat(it_wi, np.int64)
        self.max_example_items = int((ex_end - ex_start).max()) if self.nexamples else 0
        L.add("ex_item_start", ex_start)
        L.add("ex_item_end", ex_end)
        # static grouping (gm_batch.item_perm / chan_off): per example, items in
        # (output channel, item) order -- the forward's per-channel item lists
        # in the reference's accumulation order, computed once per batch
        if self.vector_mode:
            ia = L.arrays[[n for n, _ in L.arrays].index("item_atom")][1].astype(np.int64)
            ich = L.arrays[[n for n, _ in L.arrays].index("item_channel")][1].astype(np.int64)
            iset = atom_set[ia]
            chan = set_choff[iset].astype(np.int64) + ich
        else:
            iset = atom_set
            chan = set_choff[iset].astype(np.int64) + atom_type.astype(np.int64)
        C = max(self.nchannels, 1)
        key = set_example[iset].astype(np.int64) * C + chan if self.nitems else np.zeros(0, np.int64)
        # stable sort of small keys: 16-bit keys take numpy's radix sort
        skey = key.astype(np.int16) if self.nexamples * C < 32767 else key
        perm = np.argsort(skey, kind="stable").astype(np.int32)
        bounds = np.arange(self.nexamples, dtype=np.int64)[:, None] * C + \
            np.arange(self.nchannels + 1, dtype=np.int64)[None, :]
        chan_off = np.searchsorted(key[perm], bounds.reshape(-1), side="left").astype(np.int32)
        L.add("item_perm", perm)
        L.add("chan_off", chan_off)
        # groups (example * nchannels + channel) that have items (gm_batch.segs)
        segs = np.nonzero(np.diff(chan_off.reshape(self.nexamples, -1), axis=1).reshape(-1) > 0)[0] \
            if self.nexamples else np.zeros(0, np.int64)
        self.nsegs = int(segs.shape[0])
        self.max_seg_items = int(np.diff(chan_off.reshape(self.nexamples, -1), axis=1).max()) \
            if self.nexamples and self.nchannels else 0
        L.add("segs", segs.astype(np.int32))
        if not self.vector_mode and self.nitems:
            # index mode: per-slot records (gm_batch.slot_rec), item_perm order
            rec = np.zeros(self.nitems, _SLOT_DTYPE)
            a = perm.astype(np.int64)
            rec["x"], rec["y"], rec["z"] = coords[a, 0], coords[a, 1], coords[a, 2]
            rec["atom"] = a
            rec["ch"] = chan[a]
            rec["ex"] = set_example[atom_set[a]]
            rec["single"] = (counts[atom_set[a]] == 1).astype(np.int32)
            bs = self._bwd_slot_host
            rec["bslot"] = bs[a] if bs is not None else a
            rec["r"] = radius[a]
            L.add("slot_rec", rec.view(np.uint8))
        self.offsets = L.offsets

        # one pinned staging buffer -> one device buffer
        self.host = torch.empty(L.size, dtype=torch.uint8, pin_memory=self.device.type == "cuda")
        hb = self.host.numpy()
        for name, arr in L.arrays:
            off = L.offsets[name][0]
            hb[off:off + arr.nbytes] = arr.reshape(-1).view(np.uint8)
        self._to_device(L.size)

    def _to_device(self, size) -> None:
        """The device mirror of the host image (one H2D copy) and the workspace."""
        self.dev = torch.empty(size, dtype=torch.uint8, device=self.device)
        self.upload()
        nbytes = _native.lib().gm_workspace_bytes(max(self.natoms, 1), max(self.nitems, 1),
                                                   max(self.nexamples, 1), self.nchannels)
        self.workspace = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)
        self.workspace_bytes = int(nbytes)
        self._percall = None
        self._stage = None
        self._gm = None
        self._gm_ref = None

    def _pack_vector_native(self, example_sets, placed, counts, starts, scale, rti) -> None:
        """Vector typing through gm_pack_vector_host (csrc/pack.cu): the
        numpy vector packing's arrays (tested array for array), items = the
        nonzero weights atom-major then channel, the per-example launch order."""
        N, C, S, A = self.nexamples, self.nchannels, self.nsets, self.natoms
        self.default_centers = np.stack([_default_center(sets) for sets in example_sets]) \
            if N else np.zeros((0, 3))
        sets_c = (_native.GmPackVSet * max(S, 1))()
        keep, nitems, nweights, ntr = [], 0, 0, 0
        self.placed = []
        for s, (e, choff, cs) in enumerate(placed):
            n, nt = int(counts[s]), int(cs.num_types)
            ps = sets_c[s]
            ps.n, ps.example, ps.num_types = n, e, nt
            if n:
                tv = np.ascontiguousarray(cs.type_vector, np.float32)
                arrs = [np.ascontiguousarray(cs.coords, np.float32),
                        np.ascontiguousarray(cs.radii, np.float32), tv]
                if rti:
                    if cs.type_radii is None:
                        raise errors.ConfigError(
                            "radius_type_indexed requires coordinate sets typed from a table "
                            "(type_radii is missing)")
                    arrs.append(np.ascontiguousarray(cs.type_radii, np.float32))
                    ps.type_radii = arrs[3].ctypes.data
                keep.append(arrs)
                ps.coords, ps.radii, ps.type_vector = (x.ctypes.data for x in arrs[:3])
                nitems += int(np.count_nonzero(tv))
            self.placed.append((e, choff, cs, int(starts[s]), nweights))
            nweights += n * nt
            ntr += nt
        I = nitems
        order = A > 0 and _BWD_ORDER != "none"
        L = _Layout()
        L.reserve("coords32", np.float32, (A, 3))
        L.reserve("atom_radius", np.float64, (A,))
        L.reserve("atom_set", np.int32, (A,))
        for name in ("set_start", "set_end", "set_example", "set_choff", "set_t"):
            L.reserve(name, np.int32, (S,))
        if order:
            L.reserve("bwd_slot", np.int32, (A,))
        L.reserve("weights", np.float32, (nweights,))
        L.reserve("type_radius", np.float64, (ntr,))
        L.reserve("set_wstart", np.int32, (S,))
        L.reserve("set_trstart", np.int32, (S,))
        for name, dt in (("item_atom", np.int32), ("item_channel", np.int32),
                         ("item_weight", np.float32), ("item_radius", np.float64)):
            L.reserve(name, dt, (I,))
        L.reserve("ex_item_start", np.int32, (N,))
        L.reserve("ex_item_end", np.int32, (N,))
        L.reserve("item_perm", np.int32, (I,))
        L.reserve("chan_off", np.int32, (N * (C + 1),))
        L.reserve("segs", np.int32, (N * C,))
        self.host = torch.empty(L.size, dtype=torch.uint8, pin_memory=self.device.type == "cuda")
        layout = _native.GmPackVLayout(*[L.offsets[n][0] if n in L.offsets else -1
                                         for n in _native.PACK_VARRAYS])
        self.item_windex = np.empty(I, np.int64)
        centers = np.ascontiguousarray(self.default_centers, np.float64)
        info = _native.GmPackInfo()
        _native.check(_native.lib().gm_pack_vector_host(
            sets_c, S, N, C, scale, int(rti), centers.ctypes.data if N else None, int(order),
            self.host.data_ptr(), ctypes.byref(layout),
            self.item_windex.ctypes.data if I else None, ctypes.byref(info)))
        off = L.offsets["segs"][0]
        L.offsets["segs"] = (off, np.dtype(np.int32), (int(info.nsegs),))
        self.offsets = L.offsets
        self.nsegs, self.max_seg_items = int(info.nsegs), int(info.max_seg_items)
        self.max_example_items = int(info.max_example_items)
        self.nitems, self.nweights = I, nweights
        hb = self.host.numpy()
        o, dt, shape = L.offsets["atom_set"]
        atom_set = hb[o:o + A * 4].view(np.int32)
        set_example = np.array([p[0] for p in placed], np.int32)
        self.atom_example = set_example[atom_set] if A else np.zeros(0, np.int32)
        self._to_device(L.size)

    def _pack_index_native(self, example_sets, placed, counts, starts, scale) -> None:
        """Index typing: every packed array written in place, into the pinned
        host image, by the native packer (gm_pack_index_host, csrc/pack.cu) --
        the same arrays as the numpy packing (tested array for array; the
        backward launch order is a permutation with the same slab grouping)."""
        N, C, S, A = self.nexamples, self.nchannels, self.nsets, self.natoms
        self.default_centers = np.stack([_default_center(sets) for sets in example_sets]) \
            if N else np.zeros((0, 3))
        order = _BWD_ORDER == "slab" and A > 0
        L = _Layout()
        L.reserve("coords32", np.float32, (A, 3))
        L.reserve("atom_radius", np.float64, (A,))
        L.reserve("atom_set", np.int32, (A,))
        for name in ("set_start", "set_end", "set_example", "set_choff", "set_t"):
            L.reserve(name, np.int32, (S,))
        L.reserve("atom_type", np.int32, (A,))
        if order:
            L.reserve("bwd_slot", np.int32, (A,))
        L.reserve("ex_item_start", np.int32, (N,))
        L.reserve("ex_item_end", np.int32, (N,))
        L.reserve("item_perm", np.int32, (A,))
        L.reserve("chan_off", np.int32, (N * (C + 1),))
        L.reserve("segs", np.int32, (N * C,))  # capacity; the groups with items come first
        if A:
            L.reserve("slot_rec", np.uint8, (48 * A,))
        self.host = torch.empty(L.size, dtype=torch.uint8, pin_memory=self.device.type == "cuda")
        layout = _native.GmPackLayout(*[L.offsets[n][0] if n in L.offsets else -1
                                        for n in _native.PACK_ARRAYS])
        sets_c = (_native.GmPackSet * max(S, 1))()
        keep = []
        for s, (e, _, cs) in enumerate(placed):
            ps = sets_c[s]
            n = int(counts[s])
            ps.n, ps.example, ps.num_types = n, e, int(cs.num_types)
            if n:
                arrs = (np.ascontiguousarray(cs.coords, np.float32),
                        np.ascontiguousarray(cs.radii, np.float32),
                        np.ascontiguousarray(cs.type_index, np.int64))
                keep.append(arrs)
                ps.coords, ps.radii, ps.type_index = (a.ctypes.data for a in arrs)
        centers = np.ascontiguousarray(self.default_centers, np.float64)
        info = _native.GmPackInfo()
        _native.check(_native.lib().gm_pack_index_host(
            sets_c, S, N, C, scale, centers.ctypes.data if N else None, int(order),
            self.host.data_ptr(), ctypes.byref(layout), ctypes.byref(info)))
        off = L.offsets["segs"][0]
        L.offsets["segs"] = (off, np.dtype(np.int32), (int(info.nsegs),))
        self.offsets = L.offsets
        self.nsegs, self.max_seg_items = int(info.nsegs), int(info.max_seg_items)
        self.max_example_items = int(info.max_example_items)
        self.nitems, self.nweights = A, 0

        hb = self.host.numpy()

        def view(name):
            o, dt, shape = L.offsets[name]
            n = int(np.prod(shape))
            return hb[o:o + n * dt.itemsize].view(dt).reshape(shape)

        set_example = view("set_example")
        self.atom_example = set_example[view("atom_set")] if A else np.zeros(0, np.int32)
        self._bwd_slot_host = view("bwd_slot") if order else None
        self.placed = [(e, choff, cs, int(starts[s]), -1) for s, (e, choff, cs) in enumerate(placed)]
        self._to_device(L.size)

    # ------------------------------------------------------------------
    @property
    def h2d_bytes(self) -> int:
        return int(self.host.numel())

    def upload(self, non_blocking: bool = True) -> None:
        """Copy the pinned host image to the device (one H2D copy)."""
        self.dev.copy_(self.host, non_blocking=non_blocking)

    def device_view(self, name: str) -> torch.Tensor:
        """A typed tensor view of one packed array inside the device buffer."""
        off, dt, shape = self.offsets[name]
        n = int(np.prod(shape)) if len(shape) else 1
        tdt = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64,
               np.dtype(np.int32): torch.int32}[np.dtype(dt)]
        nbytes = n * np.dtype(dt).itemsize
        return self.dev[off:off + nbytes].view(tdt).view(shape)

    def load_coords(self, coords: torch.Tensor) -> None:
        """Replace the packed input-frame coordinates with a (natoms, 3)
        device tensor (a device-to-device copy, stream-ordered)."""
        if self.natoms:
            c = coords.detach().reshape(self.natoms, 3).to(torch.float32)
            self.device_view("coords32").copy_(c)
            if "slot_rec" in self.offsets:
                # index mode: the prepare pass starts from the per-slot records
                # (x, y, z gathered at pack time in item_perm order), so they
                # must follow the new coordinates too
                if getattr(self, "_perm_dev", None) is None:
                    self._perm_dev = self.device_view("item_perm").to(torch.int64)
                off = self.offsets["slot_rec"][0]
                rec = self.dev[off:off + 48 * self.nitems].view(torch.float32).view(self.nitems, 12)
                rec[:, 0:3] = c[self._perm_dev]

    def load_weights(self, weights: torch.Tensor) -> None:
        """Vector mode: replace the packed type weights (nweights,) and the
        forward items' weights.  The items (nonzero pattern) are fixed at pack
        time: entries that were zero when packed stay without a forward item."""
        if not self.vector_mode or not self.nweights:
            return
        w = weights.detach().reshape(-1).to(torch.float32)
        self.device_view("weights").copy_(w)
        if self.nitems:
            if getattr(self, "_item_windex_dev", None) is None:
                self._item_windex_dev = torch.from_numpy(self.item_windex).to(self.device)
            self.device_view("item_weight").copy_(w[self._item_windex_dev])

    def set_host_positions(self, pos: np.ndarray | None) -> None:
        """Exact-transform fallback: (natoms, 3) float64 positions already in
        the call's frame (gm_batch.coords64; the prepare pass then applies no
        transform), or None to return to device-side transforms."""
        if pos is None:
            self._want_coords64 = False
            if self._gm is not None:
                self._gm.coords64 = None
            return
        if getattr(self, "_pos64", None) is None:
            self._pos64 = torch.empty((max(self.natoms, 1), 3), dtype=torch.float64,
                                      device=self.device)
        if self.natoms:
            self._pos64[:self.natoms].copy_(torch.from_numpy(np.ascontiguousarray(pos)))
        self._want_coords64 = True
        if self._gm is not None:
            self._gm.coords64 = self._pos64.data_ptr()

    def ptr(self, name: str) -> int | None:
        if name not in self.offsets:
            return None
        return self.dev.data_ptr() + self.offsets[name][0]

    def set_call_arrays(self, origins: np.ndarray, xforms: np.ndarray | None) -> None:
        """Stage the per-call origins (N,3) and transforms (N,15), float64.

        Pinned staging slots are recycled in a ring of three, each guarded by
        an event, so the host can prepare the next call while the device
        still copies the previous one; the device-side buffer is fixed, so
        the packed ``gm_batch`` pointers never change."""
        n = self.nexamples
        cuda = self.device.type == "cuda"
        if self._percall is None:
            self._percall = torch.empty(max(18 * n, 1), dtype=torch.float64, device=self.device)
        if self._stage is None:
            self._stage = [torch.empty(max(18 * n, 1), dtype=torch.float64, pin_memory=cuda)
                           for _ in range(3)]
            self._stage_ev = [None, None, None]
            self._slot = 0
        slot = self._slot
        self._slot = (slot + 1) % 3
        if self._stage_ev[slot] is not None:
            self._stage_ev[slot].synchronize()
        h = self._stage[slot].numpy()
        h[:3 * n] = np.asarray(origins, np.float64).reshape(-1)
        m = 3 * n
        if xforms is not None:
            h[3 * n:18 * n] = np.asarray(xforms, np.float64).reshape(-1)
            m = 18 * n
        if m:
            self._percall[:m].copy_(self._stage[slot][:m], non_blocking=True)
        if cuda:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(self.device))
            self._stage_ev[slot] = ev
        self._has_xforms = xforms is not None
        if self._gm is not None:
            self._gm.xforms = self._percall.data_ptr() + 8 * 3 * n if self._has_xforms else None

    def ensure_call_buffer(self, has_xforms: bool) -> None:
        """Allocate the device per-call buffer without staging anything (the
        inline prepare path fills the origins from the launch itself)."""
        if self._percall is None:
            self._percall = torch.empty(max(18 * self.nexamples, 1), dtype=torch.float64,
                                        device=self.device)
        self._has_xforms = bool(has_xforms)
        if self._gm is not None:
            self._gm.xforms = (self._percall.data_ptr() + 8 * 3 * self.nexamples
                               if self._has_xforms else None)

    def ensure_fwd_jobs(self, params) -> None:
        """Forward job table of the static grouping for ``params.npts`` (built
        once per grid size by the C ABI, uploaded once, cached)."""
        npts = int(params.npts)
        if _NO_JOBS or self._gm is None or getattr(self, "_jobs_npts", None) == npts or \
                not self.nexamples or not self.nchannels:
            return
        # one table per grid size, kept for the batch's lifetime: a captured
        # CUDA graph (graph.GraphStep) bakes the table's pointer into its
        # forward node, so a table must never be freed while the batch lives
        if not hasattr(self, "_jobs_by_npts"):
            self._jobs_by_npts = {}
        if npts in self._jobs_by_npts:
            self._jobs, cnt = self._jobs_by_npts[npts]
            self._jobs_npts = npts
            self._gm.fwd_jobs = self._jobs.data_ptr()
            self._gm.nfwd_jobs = int(cnt)
            self._gm.fwd_jobs_npts = npts
            return
        off = self.offsets["chan_off"][0]
        n = self.nexamples * (self.nchannels + 1)
        co = np.ascontiguousarray(self.host.numpy()[off:off + 4 * n].view(np.int32))
        lib = _native.lib()
        cnt = lib.gm_forward_jobs(ctypes.byref(params), self.nexamples, self.nchannels,
                                  co.ctypes.data, None, 0)
        if cnt < 0:
            return
        jobs = np.zeros((max(cnt, 1), 4), np.int32)
        lib.gm_forward_jobs(ctypes.byref(params), self.nexamples, self.nchannels,
                            co.ctypes.data, jobs.ctypes.data, cnt)
        self._jobs = torch.from_numpy(jobs).to(self.device)
        self._jobs_by_npts[npts] = (self._jobs, int(cnt))
        self._jobs_npts = npts
        self._gm.fwd_jobs = self._jobs.data_ptr()
        self._gm.nfwd_jobs = int(cnt)
        self._gm.fwd_jobs_npts = npts

    def gm_batch(self) -> _native.GmBatch:
        """The C-ABI batch descriptor (built once; pointers are stable)."""
        if self._percall is None:
            raise RuntimeError("set_call_arrays() must run before a launch")
        if self._gm is None:
            b = _native.GmBatch()
            b.nexamples, b.nsets, b.natoms = self.nexamples, self.nsets, self.natoms
            b.nitems, b.nchannels = self.nitems, self.nchannels
            b.vector_mode = int(self.vector_mode)
            b.nweights = self.nweights
            b.max_example_items = self.max_example_items
            b.nsegs = self.nsegs
            b.max_seg_items = self.max_seg_items
            for name in ("coords32", "atom_radius", "atom_set", "atom_type", "set_start",
                         "set_end", "set_example", "set_choff", "set_t", "set_wstart", "weights",
                         "type_radius", "set_trstart", "item_atom", "item_channel",
                         "item_weight", "item_radius", "ex_item_start", "ex_item_end",
                         "item_perm", "chan_off", "bwd_slot", "slot_rec", "segs"):
                setattr(b, name, self.ptr(name))
            if getattr(self, "_want_coords64", False) and self._pos64 is not None:
                b.coords64 = self._pos64.data_ptr()
            base = self._percall.data_ptr()
            b.origins = base
            b.xforms = base + 8 * 3 * self.nexamples if self._has_xforms else None
            self._gm = b
        return self._gm


# gm_batch.slot_rec record (include/gridmaker_b200.h)
_SLOT_DTYPE = np.dtype([("x", "<f4"), ("y", "<f4"), ("z", "<f4"), ("atom", "<i4"), ("ch", "<i4"),
                        ("ex", "<i4"), ("single", "<i4"), ("bslot", "<i4"), ("r", "<f8"),
                        ("pad", "<f8")])
assert _SLOT_DTYPE.itemsize == 48

# GM_BWD_ORDER: backward launch order of the atoms -- "slab" (default: grouped
# by (example, channel) grid_grad slab, nearest the center first within a slab;
# tools/bwd_order_ab.sh: C2 94.7 us, C5 DRAM reads halved), "lpt" (heaviest
# first over the whole batch: C2 96.6 us), "lpt_local" (within examples; vector
# mode always orders within each example, C4 374 -> 349 us), "alt" (heavy /
# light alternating) or "none" (atom order)
_BWD_ORDER = os.environ.get("GM_BWD_ORDER", "slab")


def _bwd_slots(coords, atom_example, centers, per_example=False, slab=None):
    """Launch slot of each atom for the index-mode backward (gm_batch.bwd_slot).

    An atom's backward cost is its cutoff sphere's overlap with the grid, which
    falls with its distance from the example's center (rotations about the
    center preserve it).  Atoms are ranked by that distance (nearest = heaviest):
    the longest one-warp CTAs start first and the short ones fill the tail."""
    n = coords.shape[0]
    if n == 0 or _BWD_ORDER == "none":
        return None
    diff = coords - centers[atom_example].astype(np.float32)
    d2 = np.einsum("ij,ij->i", diff, diff)
    # distance in 1/16 A steps as a 16-bit key: numpy's radix sort (the order
    # only has to rank atoms by cost, ties keep atom order)
    key = np.minimum(np.sqrt(d2) * 16.0, 32767).astype(np.int16)
    # heaviest first; per_example keeps each example's atoms together (its
    # grid_grad slabs stay in L2: the vector backward reads every channel)
    per_example = per_example or _BWD_ORDER == "lpt_local"
    if per_example:
        slab = atom_example  # grouped by example, nearest first within it
    if per_example or (_BWD_ORDER == "slab" and slab is not None):
        # the atoms of one (example, channel) grid_grad slab together, nearest
        # first: overlapping spheres re-read the slab from L2 (C5 DRAM reads
        # 1152 -> 552 MB, 3.5x -> 1.7x the footprint; times unchanged).  Two
        # stable 16-bit sorts (numpy's radix sort) instead of one 64-bit sort.
        order = np.argsort(key, kind="stable")
        sl = slab[order]
        sl = sl.astype(np.int16) if sl.size and int(sl.max()) < 32767 else sl
        order = order[np.argsort(sl, kind="stable")]
        key = None
    if key is not None:
        order = np.argsort(key, kind="stable")
    if _BWD_ORDER == "alt":
        alt = np.empty(n, np.int64)
        alt[0::2] = order[:(n + 1) // 2]
        alt[1::2] = order[(n + 1) // 2:][::-1]
        order = alt
    elif _BWD_ORDER.startswith("mix:") and not per_example:
        # H atoms from the heavy end, then L from the light end, repeated
        h, l_ = (int(v) for v in _BWD_ORDER[4:].split(":"))
        out, lo, hi, k = [], 0, n, 0
        while lo < hi:
            if k % (h + l_) < h:
                out.append(order[lo])
                lo += 1
            else:
                hi -= 1
                out.append(order[hi])
            k += 1
        order = np.asarray(out, np.int64)
    slot = np.empty(n, np.int32)
    slot[order] = np.arange(n, dtype=np.int32)
    return slot


def _default_center(sets) -> np.ndarray:
    """voxelizer.py:305-309: centroid of the last non-empty set, else 0."""
    for cs in reversed(sets):
        if cs.coords.shape[0]:
            return cs.coords.astype(np.float64).mean(axis=0)
    return np.zeros(3, dtype=np.float64)


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)
_get_device = getattr(torch._C, "_cuda_getDevice", None)


def device_index(device) -> int:
    """CUDA device ordinal of ``device`` (torch.device, 'cuda:N', int; the
    current device when it names none)."""
    if isinstance(device, int):
        return device
    if not isinstance(device, torch.device):
        device = torch.device("cuda" if device is None else device)
    return device.index if device.index is not None else torch.cuda.current_device()


def stream_handle(device) -> int:
    """cudaStream_t of torch's current stream on ``device`` (the stream every
    call is ordered on).  The raw query skips the Stream object torch would
    build (a few us per call: small batches are bound by host launch work)."""
    if _raw_stream is not None:
        return _raw_stream(device_index(device))
    return torch.cuda.current_stream(device).cuda_stream


def on_device(device):
    """``torch.cuda.device(device)``, or nothing when it is already current."""
    idx = device_index(device)
    if _get_device is not None and _get_device() == idx:
        return contextlib.nullcontext()
    return torch.cuda.device(idx)


def as_ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())

"""Device-resident datasets: fresh batches assembled on the GPU (SURVEY 8(a)
row a9 and 8(f) row 1).

The reference re-packs every batch on the host: ``ExampleProvider.next_batch``
(/root/reference/pkg/src/voxmol/sampling.py:364-380) hands examples to
``GridMaker.forward_batch``, whose ``_run_batch`` concatenates the sets into
CSR arrays (voxelizer.py:372-435) before the kernels run.  Here the examples
are uploaded ONCE (``DeviceDataset``: atom records already grouped by output
channel per example, set tables, per-example channel offsets), and a batch
is just a list of example indices: ``AssembledBatch.assemble`` issues one
C-ABI call (``gm_assemble``) that builds the packed batch -- the same arrays
``PackedBatch`` uploads from the host -- and its forward job table with
sm_100a kernels, without a host sync.  The batch then goes through the usual
``GridMaker.forward_packed`` / ``backward_packed``.

Index- and vector-typed datasets (a dataset is one or the other).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native, errors
from .coordsets import coord_sets_of
from .packing import PackedBatch, _default_center, _Layout, on_device, stream_handle

# gm_dataset.records entry (include/gridmaker_b200.h)
_DS_DTYPE = np.dtype([("x", "<f4"), ("y", "<f4"), ("z", "<f4"), ("r", "<f4"), ("atom", "<i4"),
                      ("ch", "<i4"), ("brank", "<i4"), ("set_single", "<i4")])
assert _DS_DTYPE.itemsize == 32


def _local_launch_rank(coords, center):
    """Backward launch rank of each atom within its example: nearest to the
    center first (its cutoff sphere overlaps the grid most), like
    packing._bwd_slots per example."""
    diff = coords - center.astype(np.float32)
    key = np.minimum(np.sqrt(np.einsum("ij,ij->i", diff, diff)) * 16.0, 32767).astype(np.int16)
    order = np.argsort(key, kind="stable")
    rank = np.empty(coords.shape[0], np.int32)
    rank[order] = np.arange(coords.shape[0], dtype=np.int32)
    return rank


_DSI_DTYPE = np.dtype([("atom", "<i4"), ("ch", "<i4"), ("w", "<f4"), ("gpos", "<i4")])
assert _DSI_DTYPE.itemsize == 16


def _dataset_mode(example_sets):
    """None (no atoms), False (index) or True (vector) -- voxelizer.py:342-352."""
    mode = None
    for sets in example_sets:
        for cs in sets:
            if cs.coords.shape[0] == 0:
                continue
            vec = getattr(cs, "type_vector", None) is not None
            if mode is None:
                mode = vec
            elif mode != vec:
                raise ValueError("cannot mix index- and vector-typed sets in one batch")
    return mode


class DeviceDataset:
    """Examples resident in device memory, ready for ``AssembledBatch``.

    ``examples``: Examples / lists of CoordinateSets (the reference's own
    objects are accepted), every example with the same channel count, all
    index-typed or all vector-typed.  ``centers`` (per example, f64) are the
    reference defaults (voxelizer.py:305-309: centroid of the last non-empty
    set).
    """

    def __init__(self, examples, device=None):
        dev = torch.device(device) if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        example_sets = [list(ex) if isinstance(ex, (list, tuple)) else coord_sets_of(ex)
                        for ex in examples]
        if not example_sets:
            raise ValueError("a dataset needs at least one example")
        nch = {sum(int(cs.num_types) for cs in sets) for sets in example_sets}
        if len(nch) != 1:
            raise ValueError(f"examples disagree on channel count: {sorted(nch)}")
        C = nch.pop()
        if C < 1:
            raise ValueError("examples have no channels")
        self.nexamples = E = len(example_sets)
        self.nchannels = C
        self.vector_mode = bool(_dataset_mode(example_sets))
        recs, set_rows, chan_off, items, wts, trs = [], [], [], [], [], []
        ex_atom_off = np.zeros(E + 1, np.int32)
        ex_set_off = np.zeros(E + 1, np.int32)
        ex_item_off = np.zeros(E + 1, np.int32)
        ex_w_off = np.zeros(E + 1, np.int32)
        ex_tr_off = np.zeros(E + 1, np.int32)
        nzch = np.zeros(E, np.int32)
        maxch = np.zeros(E, np.int32)
        self.has_type_radii = np.ones(E, bool)
        centers = np.zeros((E, 3), np.float64)
        self.atom_counts = np.zeros(E, np.int64)
        for e, sets in enumerate(example_sets):
            counts = [int(cs.coords.shape[0]) for cs in sets]
            na = sum(counts)
            xyz = np.zeros((na, 3), np.float32)
            rad = np.zeros(na, np.float32)
            ch = np.zeros(na, np.int32)
            sset = np.zeros(na, np.int32)
            single = np.zeros(na, np.int32)
            ia_l, ic_l, iw_l, ich_l = [], [], [], []
            a = choff = woff = troff = 0
            for si, cs in enumerate(sets):
                n, nt = counts[si], int(cs.num_types)
                set_rows.append((a, n, choff, nt, woff, troff))
                if n:
                    xyz[a:a + n] = cs.coords
                    rad[a:a + n] = cs.radii
                    sset[a:a + n] = si
                    single[a:a + n] = int(n == 1)
                    if self.vector_mode:
                        tv = np.asarray(cs.type_vector, np.float32)
                        wts.append(tv.reshape(-1))
                        ia, ic = np.nonzero(tv)  # row-major: atom-major, channel-minor
                        ia_l.append(ia + a)
                        ic_l.append(ic)
                        iw_l.append(tv[ia, ic])
                        ich_l.append(ic + choff)
                        if cs.type_radii is None:
                            self.has_type_radii[e] = False
                    else:
                        ch[a:a + n] = choff + np.asarray(cs.type_index, np.int64)
                if self.vector_mode:
                    tr = getattr(cs, "type_radii", None)
                    trs.append(np.asarray(tr, np.float32) if tr is not None
                               else np.ones(nt, np.float32))
                    woff += n * nt
                    troff += nt
                a += n
                choff += nt
            centers[e] = _default_center(sets)
            brank = _local_launch_rank(xyz, centers[e])
            if self.vector_mode:
                # atoms in set order; items in item order, each with its slot in
                # the example's channel grouping
                rec = np.zeros(na, _DS_DTYPE)
                rec["x"], rec["y"], rec["z"], rec["r"] = xyz[:, 0], xyz[:, 1], xyz[:, 2], rad
                rec["atom"] = np.arange(na, dtype=np.int32)
                rec["ch"] = -1
                rec["brank"] = brank
                rec["set_single"] = sset | (single << 16)
                cat = (lambda parts, dt: np.concatenate(parts).astype(dt) if parts
                       else np.zeros(0, dt))
                ich = cat(ich_l, np.int64)
                order = np.argsort(ich, kind="stable")
                it = np.zeros(ich.shape[0], _DSI_DTYPE)
                it["atom"], it["ch"], it["w"] = cat(ia_l, np.int32), cat(ic_l, np.int32), \
                    cat(iw_l, np.float32)
                gpos = np.empty(ich.shape[0], np.int32)
                gpos[order] = np.arange(ich.shape[0], dtype=np.int32)
                it["gpos"] = gpos
                items.append(it)
                cnt = np.bincount(ich, minlength=C)[:C] if ich.shape[0] else np.zeros(C, np.int64)
                ex_item_off[e + 1] = ex_item_off[e] + ich.shape[0]
                ex_w_off[e + 1] = ex_w_off[e] + woff
                ex_tr_off[e + 1] = ex_tr_off[e] + troff
            else:
                order = np.argsort(ch, kind="stable")  # channel groups, atom order within
                rec = np.zeros(na, _DS_DTYPE)
                rec["x"], rec["y"], rec["z"] = xyz[order, 0], xyz[order, 1], xyz[order, 2]
                rec["r"] = rad[order]
                rec["atom"] = order.astype(np.int32)
                rec["ch"] = ch[order]
                rec["brank"] = brank[order]
                rec["set_single"] = sset[order] | (single[order] << 16)
                cnt = np.bincount(ch, minlength=C)[:C] if na else np.zeros(C, np.int64)
            recs.append(rec)
            co = np.zeros(C + 1, np.int32)
            co[1:] = np.cumsum(cnt)
            chan_off.append(co)
            nzch[e] = int((cnt > 0).sum())
            maxch[e] = int(cnt.max()) if cnt.shape[0] else 0
            ex_atom_off[e + 1] = ex_atom_off[e] + na
            ex_set_off[e + 1] = ex_set_off[e] + len(sets)
            self.atom_counts[e] = na
        self.centers = centers
        self.max_atoms = int(self.atom_counts.max())
        self.max_sets = int(np.diff(ex_set_off).max())
        self.max_items = int(np.diff(ex_item_off).max()) if self.vector_mode else self.max_atoms
        self.max_weights = int(np.diff(ex_w_off).max()) if self.vector_mode else 0
        self.max_type_radii = int(np.diff(ex_tr_off).max()) if self.vector_mode else 0
        self.item_counts = np.diff(ex_item_off).astype(np.int64) if self.vector_mode else \
            self.atom_counts
        rows = np.asarray(set_rows, np.int32).reshape(-1, 6)
        # host mirrors (kept alive: gm_dataset points at them)
        self._h = {"ex_atom_off": ex_atom_off, "ex_set_off": ex_set_off, "nzch": nzch,
                   "maxch": maxch, "ex_item_off": ex_item_off, "ex_w_off": ex_w_off,
                   "ex_tr_off": ex_tr_off}
        L = _Layout()
        L.add("records", np.concatenate(recs).view(np.uint8) if recs else np.zeros(32, np.uint8))
        L.add("ex_atom_off", ex_atom_off)
        L.add("ex_set_off", ex_set_off)
        L.add("ex_chan_off", np.concatenate(chan_off))
        for i, name in enumerate(("set_aoff", "set_natoms", "set_choff", "set_t", "set_woff",
                                  "set_troff")):
            L.add(name, np.ascontiguousarray(rows[:, i]))
        if self.vector_mode:
            L.add("items", np.concatenate(items).view(np.uint8) if items else np.zeros(16, np.uint8))
            L.add("weights", np.concatenate(wts) if wts else np.zeros(1, np.float32))
            L.add("type_radii", np.concatenate(trs) if trs else np.zeros(1, np.float32))
            L.add("ex_item_off", ex_item_off)
            L.add("ex_w_off", ex_w_off)
            L.add("ex_tr_off", ex_tr_off)
        host = np.zeros(L.size, np.uint8)
        for name, arr in L.arrays:
            off = L.offsets[name][0]
            host[off:off + arr.nbytes] = arr.reshape(-1).view(np.uint8)
        self.dev = torch.from_numpy(host).to(dev)
        self.nbytes = int(L.size)
        base = self.dev.data_ptr()
        d = _native.GmDataset()
        d.nexamples, d.nchannels = E, C
        d.natoms, d.nsets = int(ex_atom_off[-1]), int(ex_set_off[-1])
        for name in ("records", "ex_atom_off", "ex_set_off", "ex_chan_off", "set_aoff",
                     "set_natoms", "set_choff", "set_t", "set_woff", "set_troff"):
            setattr(d, name, base + L.offsets[name][0])
        d.h_ex_atom_off = ex_atom_off.ctypes.data
        d.h_ex_set_off = ex_set_off.ctypes.data
        d.h_ex_nzch = nzch.ctypes.data
        d.h_ex_maxch = maxch.ctypes.data
        d.vector_mode = int(self.vector_mode)
        if self.vector_mode:
            d.nitems, d.nweights = int(ex_item_off[-1]), int(ex_w_off[-1])
            d.ntype_radii = int(ex_tr_off[-1])
            for name in ("items", "weights", "type_radii", "ex_item_off", "ex_w_off", "ex_tr_off"):
                setattr(d, name, base + L.offsets[name][0])
            d.h_ex_item_off = ex_item_off.ctypes.data
            d.h_ex_w_off = ex_w_off.ctypes.data
            d.h_ex_tr_off = ex_tr_off.ctypes.data
        self._ds = d

    def batch(self, max_examples: int) -> "AssembledBatch":
        """A reusable batch of up to ``max_examples`` examples of this dataset."""
        return AssembledBatch(self, max_examples)


class AssembledBatch(PackedBatch):
    """A ``PackedBatch`` whose arrays are written on the device by
    ``gm_assemble`` from a ``DeviceDataset`` (capacity fixed at creation,
    contents replaced by every ``assemble``)."""

    def __init__(self, dataset: DeviceDataset, max_examples: int):
        if not 1 <= max_examples <= _native.INLINE_MAX_EXAMPLES:
            raise ValueError(f"max_examples must be in 1..{_native.INLINE_MAX_EXAMPLES}")
        self.dataset = dataset
        self.device = dataset.device
        self.capacity = n = int(max_examples)
        self.vector_mode = vec = dataset.vector_mode
        self.nweights = 0
        C = dataset.nchannels
        self.nchannels = C
        cap = _native.GmCapacity()
        cap.atoms = max(1, n * dataset.max_atoms)
        cap.sets = max(1, n * dataset.max_sets)
        cap.items = max(1, n * dataset.max_items)
        cap.weights = max(1, n * dataset.max_weights)
        cap.type_radii = max(1, n * dataset.max_type_radii)
        self._cap = cap
        self.atom_capacity, self.set_capacity = cap.atoms, cap.sets
        L = _Layout()
        e32 = lambda k: np.empty(k, np.int32)  # noqa: E731
        L.add("coords32", np.empty((cap.atoms, 3), np.float32))
        L.add("atom_radius", np.empty(cap.atoms, np.float64))
        L.add("atom_set", e32(cap.atoms))
        for name in ("set_start", "set_end", "set_example", "set_choff", "set_t"):
            L.add(name, e32(cap.sets))
        L.add("bwd_slot", e32(cap.atoms))
        L.add("ex_item_start", e32(n))
        L.add("ex_item_end", e32(n))
        L.add("item_perm", e32(cap.items))
        L.add("chan_off", e32(n * (C + 1)))
        L.add("segs", e32(n * C))
        if vec:
            L.add("set_wstart", e32(cap.sets))
            L.add("set_trstart", e32(cap.sets))
            L.add("weights", np.empty(cap.weights, np.float32))
            L.add("type_radius", np.empty(cap.type_radii, np.float64))
            L.add("item_atom", e32(cap.items))
            L.add("item_channel", e32(cap.items))
            L.add("item_weight", np.empty(cap.items, np.float32))
            L.add("item_radius", np.empty(cap.items, np.float64))
        else:
            L.add("atom_type", e32(cap.atoms))
            L.add("slot_rec", np.empty(cap.atoms * 48, np.uint8))
        self.offsets = L.offsets
        self.dev = torch.empty(L.size, dtype=torch.uint8, device=self.device)
        self.host = None
        with torch.cuda.device(self.device):
            nbytes = _native.lib().gm_workspace_bytes(cap.atoms, cap.items, n, C)
        self.workspace = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)
        self.workspace_bytes = int(nbytes)
        self._percall = torch.empty(18 * n, dtype=torch.float64, device=self.device)
        self._stage = None
        self._has_xforms = False
        self._jobs_cap = 0
        self._jobs = None
        b = _native.GmBatch()
        for name in L.offsets:
            setattr(b, name, self.ptr(name))
        b.nchannels = C
        b.vector_mode = int(vec)
        b.origins = self._percall.data_ptr()
        self._gm = b
        self.ids = None
        self.nexamples = self.natoms = self.nitems = self.nsets = 0

    # -- PackedBatch API -------------------------------------------------------
    @property
    def h2d_bytes(self) -> int:
        return 0 if self.ids is None else int(self.ids.nbytes)

    def upload(self, non_blocking: bool = True) -> None:
        """Nothing to upload: the batch is assembled on the device."""

    def gm_batch(self) -> _native.GmBatch:
        return self._gm

    def ensure_call_buffer(self, has_xforms: bool) -> None:
        self._has_xforms = bool(has_xforms)
        self._gm.xforms = (self._percall.data_ptr() + 8 * 3 * self.nexamples
                           if self._has_xforms else None)

    def ensure_fwd_jobs(self, params) -> None:
        if self.ids is not None and int(params.npts) != self._asm_npts:
            self._assemble(params)  # same examples, another grid size

    def load_coords(self, coords) -> None:
        """Replace the assembled batch's input-frame coordinates ((natoms, 3)
        device tensor, batch atom order) -- also in the slot records the
        index-mode prepare pass starts from."""
        if not self.natoms:
            return
        c = coords.detach().reshape(self.natoms, 3).to(torch.float32)
        self.device_view("coords32")[:self.natoms].copy_(c)
        if not self.vector_mode:
            perm = self.device_view("item_perm")[:self.nitems].to(torch.int64)
            off = self.offsets["slot_rec"][0]
            rec = self.dev[off:off + 48 * self.nitems].view(torch.float32).view(self.nitems, 12)
            rec[:, 0:3] = c[perm]

    def load_weights(self, weights) -> None:
        raise NotImplementedError("type-weight updates on device-assembled batches; "
                                  "pack the examples with GridMaker.pack for autograd weights")

    @property
    def atom_example(self) -> np.ndarray:
        counts = self.dataset.atom_counts[self.ids]
        return np.repeat(np.arange(len(self.ids), dtype=np.int32), counts)

    # -- assembly ----------------------------------------------------------------
    def assemble(self, gm, ids, stream=None) -> "AssembledBatch":
        """Make this batch the examples ``ids`` of the dataset (in that order),
        for ``gm``'s grid; stream-ordered on ``stream`` (default: the current
        stream), no host sync."""
        ids = np.ascontiguousarray(ids, dtype=np.int32).reshape(-1)
        if not 1 <= ids.shape[0] <= self.capacity:
            raise ValueError(f"batch of {ids.shape[0]} examples, capacity {self.capacity}")
        if (self.vector_mode and bool(gm.radius_type_indexed) and
                not self.dataset.has_type_radii[ids].all()):
            raise errors.ConfigError(
                "radius_type_indexed requires coordinate sets typed from a table "
                "(type_radii is missing)")
        self.ids = ids
        self.default_centers = self.dataset.centers[ids]
        self._origin_key = None  # GridMaker._prepare caches origins per batch
        self._last_params = None
        self._assemble(gm._gm_params(gm.points_per_side()), stream)
        return self

    def _job_capacity(self, params) -> int:
        """Entries for the densest table of this capacity (every group with
        items) plus the builder's 2-per-group scratch."""
        C, n = self.nchannels, self.capacity
        full = np.ones((n, C + 1), np.int32).cumsum(axis=1).astype(np.int32) - 1
        full += (np.arange(n, dtype=np.int32) * C)[:, None]
        full = np.ascontiguousarray(full)
        cnt = _native.lib().gm_forward_jobs(ctypes.byref(params), n, C, full.ctypes.data, None, 0)
        return int(cnt) + 2 * n * C

    def _assemble(self, params, stream=None) -> None:
        if self._jobs_cap == 0 or getattr(self, "_jobs_cap_npts", None) != int(params.npts):
            need = self._job_capacity(params)
            if need > self._jobs_cap:
                self._jobs = torch.empty((need, 4), dtype=torch.int32, device=self.device)
                self._jobs_cap = need
            self._jobs_cap_npts = int(params.npts)
        self._cap.jobs = self._jobs_cap
        sh = stream.cuda_stream if stream is not None else stream_handle(self.device)
        with on_device(self.device):
            _native.check(_native.lib().gm_assemble(
                ctypes.byref(params), ctypes.byref(self.dataset._ds), self.ids.ctypes.data,
                int(self.ids.shape[0]), ctypes.byref(self._gm), ctypes.byref(self._cap),
                self._jobs.data_ptr(), sh))
        g = self._gm
        self.nexamples, self.natoms, self.nitems, self.nsets = \
            g.nexamples, g.natoms, g.nitems, g.nsets
        self.nweights = g.nweights
        self.max_example_items, self.max_seg_items, self.nsegs = \
            g.max_example_items, g.max_seg_items, g.nsegs
        self._asm_npts = int(params.npts)
        self.ensure_call_buffer(self._has_xforms)


__all__ = ["DeviceDataset", "AssembledBatch"]

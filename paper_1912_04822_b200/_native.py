"""ctypes binding of the in-tree CUDA extension ``libgridmaker_b200.so``.

The extension exposes the C ABI declared in ``include/gridmaker_b200.h``.
There is no fallback: if the library is missing or no CUDA device is
visible, every gridding call raises ``DeviceError`` (the product has no CPU
path; the CPU oracle under ``oracle/`` is test infrastructure only).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import DeviceError

PKG = Path(__file__).resolve().parent
# GM_LIB: load a differently-tuned build of the same library (tools/variants.sh)
LIB_PATH = Path(os.environ.get("GM_LIB") or PKG / "libgridmaker_b200.so")

_c_int32 = ctypes.c_int32
_c_int64 = ctypes.c_int64
_c_double = ctypes.c_double
_c_size_t = ctypes.c_size_t
_vp = ctypes.c_void_p


class GmParams(ctypes.Structure):
    """Mirror of ``gm_params`` (include/gridmaker_b200.h)."""

    _fields_ = [
        ("resolution", _c_double),
        ("dimension", _c_double),
        ("radius_scale", _c_double),
        ("gaussian_radius_multiple", _c_double),
        ("radius_multiple", _c_double),
        ("npts", _c_int32),
        ("binary", _c_int32),
        ("radius_type_indexed", _c_int32),
        ("matmul_order_1", _c_int32),
        ("matmul_order_n", _c_int32),
    ]


class GmBatch(ctypes.Structure):
    """Mirror of ``gm_batch`` (device pointers as integers)."""

    _fields_ = [
        ("nexamples", _c_int32), ("nsets", _c_int32), ("natoms", _c_int32),
        ("nitems", _c_int32), ("nchannels", _c_int32), ("vector_mode", _c_int32),
        ("coords32", _vp), ("coords64", _vp), ("atom_radius", _vp), ("atom_set", _vp),
        ("atom_type", _vp),
        ("set_start", _vp), ("set_end", _vp), ("set_example", _vp), ("set_choff", _vp),
        ("set_t", _vp), ("set_wstart", _vp), ("weights", _vp), ("nweights", _c_int32),
        ("type_radius", _vp), ("set_trstart", _vp),
        ("item_atom", _vp), ("item_channel", _vp), ("item_weight", _vp), ("item_radius", _vp),
        ("ex_item_start", _vp), ("ex_item_end", _vp), ("max_example_items", _c_int32),
        ("origins", _vp), ("xforms", _vp),
        ("item_perm", _vp), ("chan_off", _vp),
        ("fwd_jobs", _vp), ("nfwd_jobs", _c_int32), ("fwd_jobs_npts", _c_int32),
        ("bwd_slot", _vp), ("slot_rec", _vp), ("segs", _vp), ("nsegs", _c_int32),
        ("max_seg_items", _c_int32),
    ]


class GmDataset(ctypes.Structure):
    """Mirror of ``gm_dataset`` (device pointers and host mirrors as integers)."""

    _fields_ = [
        ("nexamples", _c_int32), ("nchannels", _c_int32), ("natoms", _c_int32),
        ("nsets", _c_int32),
        ("records", _vp), ("ex_atom_off", _vp), ("ex_set_off", _vp), ("ex_chan_off", _vp),
        ("set_aoff", _vp), ("set_natoms", _vp), ("set_choff", _vp), ("set_t", _vp),
        ("h_ex_atom_off", _vp), ("h_ex_set_off", _vp), ("h_ex_nzch", _vp), ("h_ex_maxch", _vp),
        ("vector_mode", _c_int32), ("nitems", _c_int32), ("nweights", _c_int32),
        ("ntype_radii", _c_int32),
        ("items", _vp), ("weights", _vp), ("type_radii", _vp),
        ("ex_item_off", _vp), ("ex_w_off", _vp), ("ex_tr_off", _vp),
        ("set_woff", _vp), ("set_troff", _vp),
        ("h_ex_item_off", _vp), ("h_ex_w_off", _vp), ("h_ex_tr_off", _vp),
    ]


class GmCapacity(ctypes.Structure):
    """Mirror of ``gm_capacity``."""

    _fields_ = [("atoms", _c_int32), ("sets", _c_int32), ("items", _c_int32),
                ("weights", _c_int32), ("type_radii", _c_int32), ("jobs", _c_int32)]


class GmPackSet(ctypes.Structure):
    """Mirror of ``gm_pack_set``."""

    _fields_ = [("coords", _vp), ("radii", _vp), ("type_index", _vp), ("n", _c_int64),
                ("example", _c_int32), ("num_types", _c_int32)]


PACK_ARRAYS = ("coords32", "atom_radius", "atom_set", "atom_type", "set_start", "set_end",
               "set_example", "set_choff", "set_t", "bwd_slot", "ex_item_start", "ex_item_end",
               "item_perm", "chan_off", "segs", "slot_rec")


class GmPackLayout(ctypes.Structure):
    """Mirror of ``gm_pack_layout`` (byte offsets, -1 = absent)."""

    _fields_ = [(name, _c_int64) for name in PACK_ARRAYS]


class GmPackVSet(ctypes.Structure):
    """Mirror of ``gm_pack_vset``."""

    _fields_ = [("coords", _vp), ("radii", _vp), ("type_vector", _vp), ("type_radii", _vp),
                ("n", _c_int64), ("example", _c_int32), ("num_types", _c_int32)]


PACK_VARRAYS = ("coords32", "atom_radius", "atom_set", "set_start", "set_end", "set_example",
                "set_choff", "set_t", "set_wstart", "set_trstart", "weights", "type_radius",
                "item_atom", "item_channel", "item_weight", "item_radius", "bwd_slot",
                "ex_item_start", "ex_item_end", "item_perm", "chan_off", "segs")


class GmPackVLayout(ctypes.Structure):
    """Mirror of ``gm_pack_vlayout`` (byte offsets, -1 = absent)."""

    _fields_ = [(name, _c_int64) for name in PACK_VARRAYS]


class GmPackInfo(ctypes.Structure):
    """Mirror of ``gm_pack_info``."""

    _fields_ = [("natoms", _c_int32), ("nsegs", _c_int32), ("max_seg_items", _c_int32),
                ("max_example_items", _c_int32)]


_LIB = None
INLINE_MAX_EXAMPLES = 200  # GM_INLINE_MAX_EXAMPLES

EXPORTS = (
    "gm_workspace_bytes", "gm_prepare", "gm_prepare_inline", "gm_forward", "gm_backward", "gm_workspace_positions",
    "gm_forward_index_sets_host", "gm_forward_vector_sets_host", "gm_backward_index_host",
    "gm_backward_vector_host", "gm_last_error", "gm_version", "gm_device_count",
    "gm_launch_count", "gm_struct_size", "gm_draw_transforms", "gm_forward_jobs",
    "gm_assemble",
    "gm_molc_decode",
    "gm_pack_index_host",
    "gm_pack_vector_host",
)


def load_library(path: str | os.PathLike | None = None) -> ctypes.CDLL:
    """Load and type the extension (no device needed just to load)."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise DeviceError(
            f"CUDA extension not built: {p} is missing (run __graft_entry__.build() or "
            "make -C paper_1912_04822_b200/csrc)")
    L = ctypes.CDLL(str(p))
    P = ctypes.POINTER
    L.gm_workspace_bytes.argtypes = [_c_int32, _c_int32, _c_int32, _c_int32]
    L.gm_workspace_bytes.restype = _c_size_t
    L.gm_prepare.argtypes = [P(GmParams), P(GmBatch), _vp, _c_size_t, _vp]
    L.gm_prepare.restype = ctypes.c_int
    L.gm_prepare_inline.argtypes = [P(GmParams), P(GmBatch), _vp, _c_size_t, _vp, _vp, _vp]
    L.gm_prepare_inline.restype = ctypes.c_int
    L.gm_forward.argtypes = [P(GmParams), P(GmBatch), _vp, _vp, _vp]
    L.gm_forward.restype = ctypes.c_int
    L.gm_backward.argtypes = [P(GmParams), P(GmBatch), _vp, _vp, _vp, _vp, _vp]
    L.gm_backward.restype = ctypes.c_int
    L.gm_workspace_positions.argtypes = [_vp]
    L.gm_workspace_positions.restype = _vp
    L.gm_forward_index_sets_host.argtypes = [
        _vp, _c_int64, _c_int64, _c_int64, _vp, _vp, _vp, _c_int64, _vp, _vp, _vp, _vp, _vp,
        _c_int64, _vp, _c_double, _c_double, _c_double, _c_int32]
    L.gm_forward_index_sets_host.restype = ctypes.c_int
    L.gm_forward_vector_sets_host.argtypes = [
        _vp, _c_int64, _c_int64, _c_int64, _vp, _c_int64, _vp, _c_int64, _vp, _vp, _vp,
        _c_int64, _vp, _c_int32, _vp, _vp, _vp, _vp, _vp, _c_int64, _vp, _c_double, _c_double,
        _c_double, _c_int32]
    L.gm_forward_vector_sets_host.restype = ctypes.c_int
    L.gm_backward_index_host.argtypes = [
        _vp, _vp, _vp, _vp, _c_int64, _vp, _c_int64, _c_int64, _vp, _c_double, _c_double,
        _c_double]
    L.gm_backward_index_host.restype = ctypes.c_int
    L.gm_backward_vector_host.argtypes = [
        _vp, _vp, _vp, _vp, _vp, _c_int64, _c_int64, _vp, _c_int64, _vp, _c_int32, _vp,
        _c_double, _c_double, _c_double]
    L.gm_backward_vector_host.restype = ctypes.c_int
    L.gm_forward_jobs.argtypes = [P(GmParams), _c_int32, _c_int32, _vp, _vp, _c_int32]
    L.gm_forward_jobs.restype = _c_int32
    L.gm_assemble.argtypes = [P(GmParams), P(GmDataset), _vp, _c_int32, P(GmBatch),
                              P(GmCapacity), _vp, _vp]
    L.gm_assemble.restype = ctypes.c_int
    L.gm_pack_index_host.argtypes = [P(GmPackSet), _c_int32, _c_int32, _c_int32, _c_double,
                                     _vp, _c_int32, _vp, P(GmPackLayout), P(GmPackInfo)]
    L.gm_pack_index_host.restype = ctypes.c_int
    L.gm_pack_vector_host.argtypes = [P(GmPackVSet), _c_int32, _c_int32, _c_int32, _c_double,
                                      _c_int32, _vp, _c_int32, _vp, P(GmPackVLayout), _vp,
                                      P(GmPackInfo)]
    L.gm_pack_vector_host.restype = ctypes.c_int
    L.gm_molc_decode.argtypes = [_vp, _vp, _c_int32, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
    L.gm_molc_decode.restype = ctypes.c_int
    L.gm_draw_transforms.argtypes = [_vp, _c_int64, _c_int32, _c_double, _vp, _vp]
    L.gm_draw_transforms.restype = ctypes.c_int
    L.gm_last_error.restype = ctypes.c_char_p
    L.gm_version.restype = ctypes.c_char_p
    L.gm_device_count.restype = _c_int32
    L.gm_struct_size.argtypes = [_c_int32]
    L.gm_struct_size.restype = _c_int32
    if L.gm_struct_size(0) != ctypes.sizeof(GmParams) or \
            L.gm_struct_size(1) != ctypes.sizeof(GmBatch) or \
            L.gm_struct_size(2) != ctypes.sizeof(GmDataset) or \
            L.gm_struct_size(3) != ctypes.sizeof(GmCapacity) or \
            L.gm_struct_size(4) != ctypes.sizeof(GmPackSet) or \
            L.gm_struct_size(5) != ctypes.sizeof(GmPackLayout) or \
            L.gm_struct_size(6) != ctypes.sizeof(GmPackInfo) or \
            L.gm_struct_size(7) != ctypes.sizeof(GmPackVSet) or \
            L.gm_struct_size(8) != ctypes.sizeof(GmPackVLayout):
        raise DeviceError("ABI mismatch between _native.py and libgridmaker_b200.so")
    L.gm_launch_count.argtypes = [_c_int32]
    L.gm_launch_count.restype = _c_int64
    if path is None:
        _LIB = L
    return L


def lib() -> ctypes.CDLL:
    return load_library()


def check(status: int) -> None:
    if status != 0:
        msg = lib().gm_last_error().decode(errors="replace")
        raise DeviceError(f"gridmaker_b200 error {status}: {msg}")


def launch_count(reset: bool = False) -> int:
    return int(lib().gm_launch_count(1 if reset else 0))

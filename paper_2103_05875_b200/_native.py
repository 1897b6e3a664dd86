"""ctypes binding of ``libprobestream.so`` (the C ABI in include/probestream.h).

There is no fallback: importing the package on a machine where the library
is missing raises ``NativeLibraryError`` the first time a native entry point
is needed, and every status code is converted into the reference's exception
class.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import LayoutMismatchError, NativeLibraryError, SlotOverflowError

LIB_PATH = Path(os.environ.get("PROBESTREAM_LIB", Path(__file__).resolve().parent / "libprobestream.so"))
ABI_VERSION = 10

PS_OK = 0
PS_ERR_VALUE = -1
PS_ERR_LAYOUT = -2
PS_ERR_SLOT_OVERFLOW = -3
PS_ERR_INDEX = -4
PS_ERR_CUDA = -5
PS_ERR_WORKSPACE = -6

PS_KIND_COLOR = 0
PS_KIND_VISIBILITY = 1

PS_SHADOW_NONE = 0
PS_SHADOW_RAYS = 1
PS_SHADOW_MAP = 2

PS_DEV_SLOT_OVERFLOW = 1
PS_DEV_INDEX = 2

_vp, _i64, _i32, _f32, _f64, _sz = C.c_void_p, C.c_int64, C.c_int32, C.c_float, C.c_double, C.c_size_t
_int = C.c_int


class BvhSizes(C.Structure):
    _fields_ = [("node_count", _i64), ("tri_count", _i64), ("tri_slots", _i64),
                ("max_depth", _i64)]


class TraceParams(C.Structure):
    _fields_ = [
        ("nx", _i32), ("ny", _i32), ("nz", _i32),
        ("probe_begin", _i32), ("probe_end", _i32),
        ("origin", _f64 * 3), ("spacing", _f64 * 3),
        ("ray_dirs", _vp), ("rays_per_probe", _i32),
        ("nodes", _vp), ("bvh_width", _i32), ("tris", _vp), ("materials", _vp),
        ("light_count", _i32), ("lights", _vp),
        ("sky", _f32 * 3), ("max_distance", _f32), ("normal_bias", _f32),
        ("shadow_mode", _i32), ("shadow_map_size", _i32), ("shadow_maps", _vp),
        ("shadow_bias", _f32),
        ("shadow_texel_begin", _i64), ("shadow_texel_end", _i64), ("passes", _i32),
        ("w_color", _vp), ("w_depth", _vp), ("inv_wsum", _vp), ("w_image", _vp),
        ("hysteresis", _f32), ("irradiance_scale", _f32),
        ("irradiance", _vp), ("moments", _vp),
        ("color_atlas", _vp), ("vis_atlas", _vp),
        ("probes_per_row_color", _i32), ("probes_per_row_vis", _i32),
        ("records", _vp), ("work_counter", _vp), ("reserve_sms", _i32),
        ("ray_records", _vp),
        ("shadow_dst", _vp), ("shadow_ndst", _i32),
    ]


_SIGNATURES = {
    "ps_last_error": (C.c_char_p, []),
    "ps_abi_version": (_int, []),
    "ps_device_sm_count": (_int, []),
    "ps_pack_color": (_int, [_vp, _i64, _i64, _i64, _vp, _vp]),
    "ps_widened_width": (_i64, [_i64]),
    "ps_pack_visibility": (_int, [_vp, _i64, _i64, _i64, _vp, _vp]),
    "ps_unpack_color": (_int, [_vp, _i64, _i64, _vp, _vp]),
    "ps_unpack_visibility": (_int, [_vp, _i64, _i64, _vp, _vp]),
    "ps_temporal_delta": (_int, [_int, _vp, _vp, _i64, _i64, _vp, _vp, _vp]),
    "ps_pack_delta": (_int, [_int, _vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "ps_encode_frame_capacity": (_i64, [_i64, _i64, _int]),
    "ps_encode_workspace_bytes": (_sz, [_i64, _i64, _int]),
    "ps_encode_frame": (_int, [_int, _vp, _vp, _i64, _i64, C.c_uint32, C.c_uint32, _vp, _i64, _vp,
                               _vp, _sz, _vp]),
    "ps_decode_workspace_bytes": (_sz, [_i64, _i64]),
    "ps_decode_frame": (_int, [_int, _vp, _i64, _vp, _i64, _i64, _vp, _vp, _vp, _sz, _vp]),
    "ps_apply_entries": (_int, [_int, _vp, _i64, _i64, _vp, _vp, _i64, _vp, _i64, _vp]),
    "ps_detect_workspace_bytes": (_sz, [_i64]),
    "ps_detect_changed": (_int, [_int, _vp, _vp, _i64, _i64, _i64, _vp, _f64, _int,
                                 _vp, _vp, _vp, _vp, _sz, _vp]),
    "ps_detect_changed_range": (_int, [_int, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _vp, _f64,
                                       _int, _vp, _vp, _vp, _vp, _sz, _vp]),
    "ps_ids_to_bits": (_int, [_vp, _vp, _i64, _i64, _vp, _vp, _vp]),
    "ps_compact_workspace_bytes": (_sz, [_i64]),
    "ps_bits_to_ids": (_int, [_vp, _i64, _vp, _vp, _vp, _sz, _vp]),
    "ps_pvs_workspace_bytes": (_sz, [_i64]),
    "ps_pvs": (_int, [_vp, _i32, _vp, _vp, _vp, _i64, _vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp,
                      _vp, _vp, _vp, _sz, _vp]),
    "ps_select_workspace_bytes": (_sz, [_i64]),
    "ps_select": (_int, [_vp, _vp, _vp, _vp, _i64, _i64, _int, _i64, _int, _vp, _vp, _vp, _sz,
                         _vp]),
    "ps_assign_workspace_bytes": (_sz, [_i64, _i64]),
    "ps_assign_bits_workspace_bytes": (_sz, [_i64, _i64]),
    "ps_assign_slots_bits": (_int, [_vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                    _vp, _vp, _sz, _vp]),
    "ps_assign_slots": (_int, [_vp, _vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp,
                               _vp, _vp, _sz, _vp]),
    "ps_build_update": (_int, [_int, _vp, _i64, _i64, _vp, _vp, _i64, _i64, _vp, _i64, _vp,
                               _vp, _i64, _vp, _vp]),
    "ps_reconstruct_guard_bands": (_int, [_int, _vp, _i64, _i64, _vp]),
    "ps_index_workspace_bytes": (_sz, [_i64]),
    "ps_encode_index": (_int, [_vp, _vp, _i64, _vp, _vp, _vp, _sz, _vp]),
    "ps_frame_advance": (_int, [_vp, _i64, _vp]),
    "ps_trace_stats": (_int, [_vp]),
    "ps_detect_changed_bcast": (_int, [_int, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _vp, _f64,
                                       _int, _vp, _int, _vp]),
    "ps_export_tiles_peer": (_int, [_int, _vp, _i64, _i64, _vp, _vp, _i64, _i64, _i64, _i64, _vp,
                                    _i64, _vp, _vp, _i64, _vp, _vp]),
    "ps_peer_signal": (_int, [_vp, _i32, _i64, _vp, _i64, _vp]),
    "ps_peer_wait": (_int, [_vp, _i32, _i64, _vp, _i64, _vp, _i64, _vp]),
    "ps_peer_status": (_int, [_vp]),
    "ps_ipc_handle_bytes": (_sz, []),
    "ps_ipc_export": (_int, [_vp, _vp, _vp]),
    "ps_ipc_open": (_int, [_vp, _i64, _vp]),
    "ps_export_tiles": (_int, [_int, _vp, _i64, _i64, _vp, _vp, _i64, _i64, _i64, _vp, _vp, _vp,
                               _i64, _vp, _vp]),
    "ps_import_tiles": (_int, [_int, _vp, _i64, _vp, _i32, _vp, _vp, _i64, _i64, _vp, _i64, _vp]),
    "ps_bvh_build": (_int, [_vp, _i64, _int, C.POINTER(BvhSizes), _vp, _vp]),
    "ps_bvh_build_wide": (_int, [_vp, _i64, _int, _int, C.POINTER(BvhSizes), _vp, _vp]),
    "ps_blend_weights": (_int, [_vp, _i32, _vp, _f32, _vp, _vp, _vp, _vp, _vp]),
    "ps_blend_weight_image_floats": (_sz, [_i32]),
    "ps_trace_blend": (_int, [C.POINTER(TraceParams), _vp]),
}

_PENDING: set = set()

_lib = None
_lock = threading.Lock()


def lib():
    """The loaded library (loads on first use; raises if it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise NativeLibraryError(
                f"{LIB_PATH} not found: build it with "
                "`python -m paper_2103_05875_b200.build_native` (no CPU fallback exists)")
        handle = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(handle, name, None)
            if fn is None:
                if name in _PENDING:
                    continue
                raise NativeLibraryError(f"{LIB_PATH} does not export {name}")
            fn.restype = res
            fn.argtypes = args
        if handle.ps_abi_version() != ABI_VERSION:
            raise NativeLibraryError("libprobestream ABI version mismatch; rebuild")
        _lib = handle
        return _lib


def exported_symbols():
    return list(_SIGNATURES)


def check(status: int, what: str = "") -> None:
    if status == PS_OK:
        return
    msg = lib().ps_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status == PS_ERR_LAYOUT:
        raise LayoutMismatchError(text)
    if status == PS_ERR_SLOT_OVERFLOW:
        raise SlotOverflowError(text)
    if status == PS_ERR_INDEX:
        raise IndexError(text)
    if status in (PS_ERR_VALUE, PS_ERR_WORKSPACE):
        raise ValueError(text)
    raise RuntimeError(text)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)

"""ctypes binding of the sm_100a C-ABI (include/respa_b200.h).

This is the whole bridge between the Python mirror of the reference API and
the CUDA kernels: device buffers are torch CUDA tensors (plumbing only),
passed by ``data_ptr()``; streams are torch streams passed by handle.

There is no fallback: if the shared library is missing or no CUDA device is
visible, :func:`lib` / :func:`require_device` raise.
"""

from __future__ import annotations

import ctypes
import os

from . import build as _build

RB_OK = 0
RB_ERR_MIN_SEPARATION = 1
RB_ERR_GEOMETRY = 2
RB_ERR_CUDA = 3
RB_ERR_CAPACITY = 4
RB_ERR_ARGUMENT = 5
RB_NOT_CAPTURING = 6

RB_KIND_PAIR_MIN_SEPARATION = 1
RB_KIND_TRIPLET_MIN_SEPARATION = 2
RB_KIND_NONFINITE = 3
RB_KIND_CAPACITY = 4
RB_KIND_REBUILD = 0  # not an error: a speculative window froze (domain loop)
RB_STATUS_CLEAR = 0xFFFFFFFFFFFFFFFF
RB_TAG_FROM_DEVICE = -1
RB_MAX_OFFSETS = 125

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_D = ctypes.c_double
_SZ = ctypes.c_size_t
_U64 = ctypes.c_uint64


class RbGrid(ctypes.Structure):
    """Mirror of ``rb_grid`` (include/respa_b200.h)."""

    _fields_ = [
        ("cells", _I32 * 3),
        ("periodic", _I32),
        ("origin", _D * 3),
        ("inv_cell", _D * 3),
        ("box", _D * 3),
        ("n_offsets", _I32),
        ("offsets", (_I32 * 3) * RB_MAX_OFFSETS),
        ("wrap", _I32 * 3),
        ("gcells", _I32 * 3),
        ("wlo", _I32 * 3),
    ]


# name -> (restype, argtypes); every symbol declared in include/respa_b200.h
SIGNATURES = {
    "rb_abi_version": (ctypes.c_int, []),
    "rb_grid_bytes": (_SZ, []),
    "rb_launch_count": (ctypes.c_longlong, []),
    "rb_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "rb_device_count": (ctypes.c_int, []),
    "rb_bin_scratch_bytes": (_SZ, [_I64, _I64]),
    "rb_bin": (ctypes.c_int, [ctypes.POINTER(RbGrid), _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _P, _SZ, _P]),
    "rb_nlist": (ctypes.c_int, [ctypes.POINTER(RbGrid), _I64, _P, _P, _P, _D, _I32, _P, _P, _P, _P, _P, _I64, _P]),
    "rb_nlist_mirror": (ctypes.c_int, [_I64, _P, _P, _I32, _P, _P, _P, _I64, _P]),
    "rb_nlist_mirror_scratch_bytes": (ctypes.c_size_t, [_I64]),
    "rb_nlist_rows_mirror": (ctypes.c_int, [ctypes.POINTER(RbGrid), _I64, _P, _P, _P, _D, _I32, _P, _P, _P, _P, _P, ctypes.c_size_t, _P, _P, _I64, _P]),
    "rb_lj_pass": (ctypes.c_int, [ctypes.POINTER(RbGrid), _I64, _P, _P, _P, _P, _I32, _D, _D, _D, _P, _P, _P, _P,
                                  _P, _I64, _P]),
    "rb_atm_scratch_bytes": (_SZ, [_I64, _I32]),
    "rb_atm_pass": (ctypes.c_int, [ctypes.POINTER(RbGrid), _I64, _P, _P, _P, _P, _P, _I32, _I32, _D, _D, _P, _P, _P, _P,
                                   _P, _P, _SZ, _P, _I64, _P]),
    "rb_atm_pass_part": (ctypes.c_int, [ctypes.POINTER(RbGrid), _I64, _P, _P, _P, _P, _P, _I32, _I32, _D, _D, _P, _P, _P, _P,
                                   _P, _P, _SZ, _P, _I64, _I32, _P]),
    "rb_atm_cells_scratch_bytes": (_SZ, [_I64]),
    "rb_atm_cells_smem_bytes": (_SZ, [_I32, _I32]),
    "rb_atm_cells_supported": (ctypes.c_int, [ctypes.POINTER(RbGrid), _D]),
    "rb_atm_cells_nb_max": (ctypes.c_int, [ctypes.POINTER(RbGrid), _P, _P, _P]),
    "rb_atm_pass_cells": (ctypes.c_int, [ctypes.POINTER(RbGrid), _I64, _P, _P, _P, _P, _I32, _I32, _D, _D, _P,
                                         _P, _P, _P, _P, _P, _SZ, _P, _I64, _I32, _P]),
    "rb_atm_pass_c01": (ctypes.c_int, [ctypes.POINTER(RbGrid), _I64, _P, _P, _P, _P, _I32, _D, _D, _P, _P, _P, _P, _P,
                                       _I64, _P]),
    "rb_atm_visit_rows": (ctypes.c_int, [ctypes.POINTER(RbGrid), _I64, _P, _P, _P, _P, _I32, _D, _P, _P, _P]),
    "rb_reduce_scratch_bytes": (_SZ, [_I64]),
    "rb_reduce_sum_f64": (ctypes.c_int, [_I64, _P, _P, _P, _P]),
    "rb_reduce_sumsq_f64": (ctypes.c_int, [_I64, _P, _P, _P, _P]),
    "rb_reduce_sum_i32": (ctypes.c_int, [_I64, _P, _P, _P, _P]),
    "rb_respa_drift": (ctypes.c_int, [_I64, _P, _P, _P, _P, _P, _I32, _D, _D, _D, _I32, _P, _P, _P, _D,
                                      _P, _P, _I64, _I32, _U64, _P]),
    "rb_respa_kick_drift": (ctypes.c_int, [_I64, _P, _P, _P, _P, _P, _P, _I32, _D, _D, _D, _D,
                                           _I32, _I32, _P, _P, _P, _D, _P, _P, _U64, _P]),
    "rb_respa_kick": (ctypes.c_int, [_I64, _P, _P, _P, _P, _D, _D, _I32, _P, _I64, _P]),
    "rb_vote_flag": (ctypes.c_int, [_P, _P, _P, _P]),
    "rb_vote_freeze": (ctypes.c_int, [_P, _P, _P]),
    "rb_step_begin": (ctypes.c_int, [_P, _P]),
    "rb_trace_record": (ctypes.c_int, [_P, _I64, _P, _P, _P, _P, _P, _P, _P]),
    "rb_fp64_peak": (ctypes.c_int, [_I32, _P, _P]),
    "rb_l2_flush": (ctypes.c_int, [_P, _SZ, _P]),
    "rb_event_create": (ctypes.c_int, [_P]),
    "rb_event_destroy": (ctypes.c_int, [_P]),
    "rb_event_record": (ctypes.c_int, [_P, _P]),
    "rb_event_elapsed": (ctypes.c_int, [_P, _P, _P]),
    "rb_direct_pairs": (ctypes.c_int, [_I64, _P, _D, _D, _P, _P, _P, _P, _I64, _P]),
    "rb_direct_scratch_bytes": (ctypes.c_size_t, [_I64]),
    "rb_direct_triplets": (ctypes.c_int, [_I64, _P, _D, _P, _P, _P, _SZ, _P, _I64, _P]),
    "rb_distance_histogram": (ctypes.c_int, [_I64, _P, _P, _D, _D, _I32, _P, _P]),
    "rb_halo_pack": (ctypes.c_int, [_I64, _P, _P, _P, _P]),
    "rb_halo_unpack": (ctypes.c_int, [_I64, _P, _I64, _P, _P, _P, _P]),
    "rb_respa_drift_publish": (ctypes.c_int, [_I64, _P, _P, _P, _P, _P, _I32, _D, _D, _D, _I32,
                                              _P, _P, _P, _D, _P, _P, _I64, _I32, _P, _I64,
                                              _P]),
    "rb_halo_pull": (ctypes.c_int, [_I64, _P, _P, _P, _I64, _P, _I64, _P, _P, _P, _P]),
    "rb_ipc_alloc": (ctypes.c_int, [_I64, ctypes.POINTER(ctypes.c_void_p)]),
    "rb_ipc_free": (ctypes.c_int, [_P]),
    "rb_ipc_handle": (ctypes.c_int, [_P, _P]),
    "rb_ipc_open": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_void_p)]),
    "rb_ipc_close": (ctypes.c_int, [_P]),
    "rb_direct_pairs_range": (ctypes.c_int, [_I64, _P, _I64, _I64, _D, _D, _P, _P, _P, _P, _I64,
                                             _P]),
    "rb_direct_triplets_range": (ctypes.c_int, [_I64, _P, _I64, _I64, _D, _P, _P, _P, _SZ, _P,
                                                _I64, _P]),
    "rb_sample_scratch_bytes": (ctypes.c_size_t, [_I64]),
    "rb_sample": (ctypes.c_int, [_I64, _P, _P, _P, _P, _P, _P, _P, _I64, _P, _P, _SZ, _P]),
    "rb_rebuild_cond_create": (ctypes.c_int, [_P, _P]),
    "rb_rebuild_cond_begin": (ctypes.c_int, [_U64, _P, _P]),
    "rb_rebuild_cond_end": (ctypes.c_int, [_P]),
    "rb_rebuild_scratch_bytes": (ctypes.c_size_t, [_I64, _I64]),
    "rb_rebuild": (ctypes.c_int, [_P, _I64, _P, _P, _P, _P, _P, _P, _P, _D, _I32, _P, _P, _P, _P,
                                  _P, _P, _I64, _P, _SZ, _P]),
    "rb_graph_begin": (ctypes.c_int, [_P]),
    "rb_graph_end": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_uint64)]),
    "rb_graph_launch": (ctypes.c_int, [_U64, _P]),
    "rb_graph_destroy": (ctypes.c_int, [_U64]),
}

_lib = None


class NativeLibraryError(RuntimeError):
    """The sm_100a library is missing, stale, or cannot run here."""


def lib():
    """Load (building in-tree first if needed) the C-ABI library."""
    global _lib
    if _lib is not None:
        return _lib
    override = os.environ.get("RB_LIB_PATH")  # tuning builds (tools/); never a fallback
    path = override or _build.LIB_PATH
    if override is None and not _build.up_to_date():
        try:
            _build.build()
        except Exception as exc:  # pragma: no cover - build environment problem
            if not os.path.exists(path):
                raise NativeLibraryError(f"sm_100a library not built and build failed: {exc}") from exc
    if not os.path.exists(path):
        raise NativeLibraryError(f"sm_100a library not found at {path}")
    L = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    if L.rb_abi_version() != 1:
        raise NativeLibraryError("ABI version mismatch")
    if L.rb_grid_bytes() != ctypes.sizeof(RbGrid):
        raise NativeLibraryError("rb_grid layout mismatch between header and binding")
    _lib = L
    return _lib


def check(status: int, what: str) -> None:
    if status != RB_OK:
        msg = lib().rb_status_string(int(status)).decode()
        raise NativeLibraryError(f"{what} failed: {msg} ({status})")


def require_device():
    """Return torch with a visible CUDA device, or raise (no CPU fallback)."""
    import torch

    if not torch.cuda.is_available():
        raise NativeLibraryError(
            "paper_2507_11172_b200 runs only on a CUDA device (sm_100a); none is visible"
        )
    if lib().rb_device_count() < 1:
        raise NativeLibraryError("the sm_100a library sees no CUDA device")
    return torch


def ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def stream_handle(stream=None) -> ctypes.c_void_p:
    import torch

    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)

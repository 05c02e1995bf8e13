"""ctypes binding of the in-tree C-ABI library ``libglint_b200.so``.

This is the only place Python touches the native boundary declared in
``include/glint_b200.h``.  There is no fallback: if the library is missing or
was not built for this GPU every call raises ``InternalError``.  Pointers are
raw CUDA device addresses (``torch.Tensor.data_ptr()``), streams are the raw
``cudaStream_t`` of the torch stream in use.
"""

from __future__ import annotations

import ctypes
import os
import pathlib
import threading

from .errors import InternalError

LIB_PATH = pathlib.Path(__file__).resolve().with_name("libglint_b200.so")
if os.environ.get("GLINT_LIB_PATH"):   # A/B builds of the same library (tools only)
    LIB_PATH = pathlib.Path(os.environ["GLINT_LIB_PATH"]).resolve()
HEADER_PATH = pathlib.Path(__file__).resolve().parents[1] / "include" / "glint_b200.h"

GLINT_OK = 0
GLINT_EINVAL = -1
GLINT_ECUDA = -2
GLINT_EUNSUPPORTED = -3

EW_KINDS = {"ReLU": 0, "LeakyReLU": 1, "Add": 2, "Norm": 3, "DropoutIdentity": 4}
ACT_NONE, ACT_RELU, ACT_LEAKY_RELU = 0, 1, 2
PREC_FP32, PREC_3XTF32 = 0, 1

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_F32 = ctypes.c_float
_SZ = ctypes.c_size_t

# name -> (restype, argtypes); the single source of the Python-side ABI.
SIGNATURES = {
    "glint_last_error": (ctypes.c_char_p, []),
    "glint_abi_version": (ctypes.c_int, []),
    "glint_set_tuning": (ctypes.c_int, [ctypes.c_int, ctypes.c_int]),
    "glint_get_tuning": (ctypes.c_int, [ctypes.c_int]),
    "glint_debug_counters": (ctypes.c_int, [ctypes.c_int, _P, ctypes.c_int, ctypes.c_int]),
    "glint_device_info": (ctypes.c_int, [ctypes.c_int, _P, _P, _P, _P, _P]),
    "glint_spmm_mean_f32": (ctypes.c_int, [_I64, _I32, _P, _P, _P, _I64, _P, _P, _P, _I64,
                                           _P, _I64, _P, _I64, _P, _I32, _P]),
    "glint_conv_mean_workspace_bytes": (_SZ, [_I32, _I32]),
    "glint_conv_mean_supported": (ctypes.c_int, [_I32, _I32]),
    "glint_conv_mean_f32": (ctypes.c_int, [_I64, _I32, _I32, _P, _P, _P, _I64, _P, _P, _P, _I64,
                                           _P, _I64, _P, _I32, _P, _I64, _P, _I32, _P, _SZ, _P]),
    "glint_degree_schedule_workspace_bytes": (_SZ, []),
    "glint_degree_schedule": (ctypes.c_int, [_I64, _P, _P, _I64, _I64, _P, _P, _P, _SZ, _P]),
    "glint_linear_f32": (ctypes.c_int, [_I64, _I32, _I32, _P, _I64, _P, _P, _I64, _P, _I32,
                                        _P, _I64, _I32, _P]),
    "glint_gat_scores_f32": (ctypes.c_int, [_I64, _I32, _I32, _I32, _P, _I64, _P, _P, _P, _P]),
    "glint_gat_project_f32": (ctypes.c_int, [_I64, _I32, _I32, _I32, _I32, _P, _I64, _P, _P,
                                             _I64, _P, _P, _I64, _P, _P, _I32, _P]),
    "glint_gat_aggregate_f32": (ctypes.c_int, [_I64, _I32, _I32, _I32, _P, _P, _P, _I64, _P,
                                               _P, _P, _I64, _P, _P, _F32, _P, _I64, _P, _I64,
                                               _I32, _P]),
    "glint_gat_aggregate_workspace_bytes": (_SZ, [_I64, _I64, _I32]),
    "glint_gat_aggregate_ws_f32": (ctypes.c_int, [_I64, _I32, _I32, _I32, _P, _P, _P, _I64, _P,
                                                  _P, _P, _I64, _P, _P, _F32, _P, _I64, _P, _I64,
                                                  _I32, _I64, _I64, _P, _SZ, _P]),
    "glint_elementwise_f32": (ctypes.c_int, [_I32, _I64, _I32, _I32, _P, _P, _P, _P, _I64, _P]),
    "glint_copy_rows_f32": (ctypes.c_int, [_I64, _I32, _P, _I64, _P, _P, _I64, _P, _P]),
    "glint_idset_workspace_bytes": (_SZ, [_I64]),
    "glint_idset_clear": (ctypes.c_int, [_P, _I64, _P]),
    "glint_idset_add_ids": (ctypes.c_int, [_P, _I64, _P, _I64, _I64, _P]),
    "glint_idset_add_neighbors": (ctypes.c_int, [_P, _I64, _P, _P, _P, _I64, _I64, _P]),
    "glint_idset_finalize": (ctypes.c_int, [_P, _I64, _P, _P]),
    "glint_idset_extract": (ctypes.c_int, [_P, _I64, _P, _P]),
    "glint_idset_lookup": (ctypes.c_int, [_P, _I64, _P, _P, _I64, _P, _P, _P]),
    "glint_idset_rank_map": (ctypes.c_int, [_P, _I64, _P, _P]),
    "glint_scan_workspace_bytes": (_SZ, [_I64]),
    "glint_degree_prefix": (ctypes.c_int, [_P, _P, _I64, _I64, _P, _P, _SZ, _P]),
    "glint_hub_prefix": (ctypes.c_int, [_P, _P, _I64, _I64, _I64, _P, _P, _SZ, _P]),
    "glint_gather_slices": (ctypes.c_int, [_P, _P, _P, _I64, _I64, _P, _P, _P, _P, _I64, _P,
                                           _P, _P]),
    "glint_relabel_csc": (ctypes.c_int, [_I64, _P, _P, _P, _P, _P, _P, _P]),
    "glint_narrow_ids": (ctypes.c_int, [_I64, _P, _P, _I64, _P, _P]),
    "glint_rcmk_host": (ctypes.c_int, [_I64, _P, _P, _P]),
    "glint_rcmk_components": (ctypes.c_int, [_I64, _P, _P, _P, _P]),
    "glint_rcmk_starts": (ctypes.c_int, [_I64, _P, _P, _P, _P]),
    "glint_rcmk_expand": (ctypes.c_int, [_I64, _P, _P, _P, _P, _P, _P]),
    "glint_rcmk_sorted_host": (ctypes.c_int, [_I64, _P, _P, _P]),
    "glint_narrow_ids_host": (_I64, [_P, _P, _I64, _I32]),
    "glint_upload_start": (ctypes.c_int, [_P, _P, _P, _P, _I32, _I32, _P, _P]),
    "glint_upload_start_packed": (ctypes.c_int, [_P, _P, _P, _P, _I32, _P, _I32, _I32, _P, _P]),
    "glint_upload_wait": (ctypes.c_int, [_P, _I32, _P]),
    "glint_copy_rows_async": (ctypes.c_int, [_P, _I64, _P, _I64, _I64, _I64, _P]),
    "glint_upload_query": (ctypes.c_int, [_P, _I32]),
    "glint_upload_finish": (ctypes.c_int, [_P]),
    "glint_h2d_pageable": (ctypes.c_int, [_P, _P, _I64, _I32, _P]),
    "glint_sample_workspace_bytes": (_SZ, [_I64, _I64, _I64]),
    "glint_sample_neighbors": (ctypes.c_int, [_P, _P, _P, _I64, _P, _I64, _P, _I64, _I32, _I64,
                                              _I32, _P, _P, _SZ, _P]),
}

_lock = threading.Lock()
_lib = None


def load():
    """Load (once) and return the ctypes library; raises InternalError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise InternalError(
                    f"native library {LIB_PATH} is missing; build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback)")
            lib = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def last_error() -> str:
    msg = load().glint_last_error()
    return msg.decode(errors="replace") if msg else ""


# Kernels launched per call (for the bench's launch count); host-only or
# memset-only entry points launch none.
KERNELS_PER_CALL = {"glint_conv_mean_f32": 2, "glint_rcmk_components": 3, "glint_degree_schedule": 3, "glint_idset_finalize": 4,
                    "glint_degree_prefix": 3, "glint_hub_prefix": 3, "glint_idset_clear": 0, "glint_rcmk_host": 0,
                    "glint_rcmk_sorted_host": 0, "glint_sample_neighbors": 4,
                    "glint_gat_aggregate_ws_f32": 2, "glint_upload_start": 0, "glint_upload_start_packed": 1, "glint_copy_rows_async": 0,
                    "glint_upload_wait": 0, "glint_upload_query": 0, "glint_upload_finish": 0,
                    "glint_h2d_pageable": 0,
                    "glint_device_info": 0, "glint_set_tuning": 0, "glint_debug_counters": 0}
LAUNCHES = [0]


def call(name, *args):
    """Invoke an int-returning entry point and map its status to an exception."""
    LAUNCHES[0] += KERNELS_PER_CALL.get(name, 1)
    rc = getattr(load(), name)(*args)
    if rc == GLINT_OK:
        return
    msg = f"{name}: {last_error()}"
    if rc == GLINT_EINVAL:
        raise ValueError(msg)
    raise InternalError(msg)


def query(name, *args):
    """Invoke a value-returning entry point (sizes, versions)."""
    return getattr(load(), name)(*args)

"""ctypes binding of the C ABI in include/patfft_b200.h.

This is the shim the drop-in ``reconstruct_nedner`` dispatches through.  It
loads the in-tree ``libpatfft_b200.so`` (built by ``_build.py``); there is
no CPU fallback -- a missing library or a CUDA failure raises DeviceError.
"""

from __future__ import annotations

import ctypes
import os
import re

from .errors import DataValidationError, DeviceError, ParameterError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PATFFT_LIB") or os.path.join(HERE, "libpatfft_b200.so")  # PATFFT_LIB: experimental variant builds
HEADER = os.path.join(os.path.dirname(HERE), "include", "patfft_b200.h")

PATFFT_OK = 0
PATFFT_ERR_PARAMETER = 1
PATFFT_ERR_DATA = 2
PATFFT_ERR_CUDA = 3
PATFFT_ERR_UNSUPPORTED = 4
N_STAGES = 5


class NednerDesc(ctypes.Structure):
    _fields_ = [
        ("n_lat", ctypes.c_int32),
        ("out_dims", ctypes.c_int32 * 2),
        ("n_time", ctypes.c_int32),
        ("upsample", ctypes.c_int32),
        ("n_sensors", ctypes.c_int32),
        ("lat_ratio", ctypes.c_double * 2),
        ("spec_c", ctypes.c_double),
        ("spec_K", ctypes.c_int32),
        ("spec_alpha", ctypes.c_double),
        ("spec_beta", ctypes.c_double),
    ]


_P = ctypes.c_void_p
_D = ctypes.POINTER(ctypes.c_double)
_SIGS = {
    "patfft_nedner_plan_create": (ctypes.c_int, [ctypes.POINTER(NednerDesc), _D, _D, ctypes.c_int, ctypes.POINTER(_P)]),
    "patfft_equispaced_plan_create": (ctypes.c_int, [ctypes.POINTER(NednerDesc), ctypes.POINTER(ctypes.c_int64),
                                                     ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)]),
    "patfft_nedner_output_shape": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int64)]),
    "patfft_nedner_execute": (ctypes.c_int, [_P, _P, _P, _D]),
    "patfft_nedner_execute_checked": (ctypes.c_int, [_P, _P, _P, _D, ctypes.POINTER(ctypes.c_int64)]),
    "patfft_nedner_execute_batch": (ctypes.c_int, [_P, ctypes.c_int, ctypes.POINTER(_P), ctypes.POINTER(_P),
                                                   ctypes.POINTER(ctypes.c_int64)]),
    "patfft_nedner_execute_device": (ctypes.c_int, [_P, _P, _P, _P]),
    "patfft_nedner_execute_frames_device": (ctypes.c_int, [_P, ctypes.c_int, _P, _P, _P]),
    "patfft_nedner_plan_destroy": (None, [_P]),
    "patfft_nedner_plan_create_sharded": (ctypes.c_int, [ctypes.POINTER(NednerDesc), _D, _D, ctypes.c_int, ctypes.c_int,
                                                         ctypes.c_int, ctypes.POINTER(_P)]),
    "patfft_nedner_shard_info": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int64)]),
    "patfft_nedner_shard_rows": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int64), ctypes.c_int]),
    "patfft_nedner_shard_forward": (ctypes.c_int, [_P, _P, _P, _P]),
    "patfft_nedner_shard_ner": (ctypes.c_int, [_P, _P, _P, _P]),
    "patfft_nedner_shard_inverse": (ctypes.c_int, [_P, _P, _P, _P]),
    "patfft_nedner_shard_spread": (ctypes.c_int, [_P, _P, _P]),
    "patfft_nedner_shard_lateral": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, _P, _P]),
    "patfft_nedner_shard_ner_rows": (ctypes.c_int, [_P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, _P]),
    "patfft_nedner_plan_create_slice": (ctypes.c_int, [ctypes.POINTER(NednerDesc), _D, _D, ctypes.c_int, ctypes.c_int,
                                                       ctypes.POINTER(_P)]),
    "patfft_nedner_slice_ner": (ctypes.c_int, [_P, _P, ctypes.c_int, ctypes.c_int, _P, _P]),
    "patfft_ner_plan_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_double,
                                              ctypes.c_double, ctypes.c_int, ctypes.POINTER(_P)]),
    "patfft_ner_plan_info": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int64)]),
    "patfft_ner_execute": (ctypes.c_int, [_P, _P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P]),
    "patfft_ner_execute_device": (ctypes.c_int, [_P, _P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, _P]),
    "patfft_ner_plan_destroy": (None, [_P]),
    "patfft_ned_plan_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_int32), ctypes.c_int,
                                              ctypes.c_double, ctypes.c_int, ctypes.c_double, ctypes.c_double, _D,
                                              ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)]),
    "patfft_ned_execute": (ctypes.c_int, [_P, _P, _P, ctypes.c_int]),
    "patfft_forward_plan_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_int32), ctypes.c_int, _D,
                                                  ctypes.c_double, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                                  ctypes.c_int, ctypes.POINTER(_P)]),
    "patfft_forward_execute": (ctypes.c_int, [_P, _P, _P]),
    "patfft_forward_execute_device": (ctypes.c_int, [_P, _P, _P, _P]),
    "patfft_forward_plan_destroy": (None, [_P]),
    "patfft_nedner_set_profiling": (ctypes.c_int, [_P, ctypes.c_int]),
    "patfft_nedner_stage_times": (ctypes.c_int, [_P, _D, ctypes.POINTER(ctypes.c_int64), ctypes.c_int]),
    "patfft_nedner_stage_name": (ctypes.c_char_p, [ctypes.c_int]),
    "patfft_nedner_stage_bytes": (ctypes.c_int, [_P, _D, ctypes.c_int]),
    "patfft_nedner_launches_per_execute": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    "patfft_nedner_spread_info": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int64)]),
    "patfft_nedner_window_info": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int64), _D]),
    "patfft_last_error": (ctypes.c_char_p, []),
    "patfft_version": (ctypes.c_char_p, []),
    "patfft_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "patfft_device_alloc": (ctypes.c_int, [ctypes.c_int, ctypes.c_size_t, ctypes.POINTER(_P)]),
    "patfft_device_free": (ctypes.c_int, [_P]),
    "patfft_host_alloc": (ctypes.c_int, [ctypes.c_size_t, ctypes.POINTER(_P)]),
    "patfft_host_free": (ctypes.c_int, [_P]),
    "patfft_memcpy_h2d": (ctypes.c_int, [_P, _P, ctypes.c_size_t, _P]),
    "patfft_memcpy_d2h": (ctypes.c_int, [_P, _P, ctypes.c_size_t, _P]),
    "patfft_stream_sync": (ctypes.c_int, [_P]),
    "patfft_plan_stream": (ctypes.c_int, [_P, ctypes.POINTER(_P)]),
    "patfft_convert_f64_to_f32": (ctypes.c_int, [_P, _P, ctypes.c_size_t, _P]),
    "patfft_convert_f32_to_f64": (ctypes.c_int, [_P, _P, ctypes.c_size_t, _P]),
    "patfft_l2_flush": (ctypes.c_int, [_P, ctypes.c_size_t, _P]),
    "patfft_event_create": (ctypes.c_int, [ctypes.POINTER(_P)]),
    "patfft_event_record": (ctypes.c_int, [_P, _P]),
    "patfft_event_elapsed_ms": (ctypes.c_int, [_P, _P, ctypes.POINTER(ctypes.c_float)]),
    "patfft_event_destroy": (ctypes.c_int, [_P]),
}

_lib = None


def header_symbols(path: str = HEADER) -> list[str]:
    """Function names declared in the public header."""
    text = open(path).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(patfft_[a-z0-9_]+)\s*\(", text)))


def load():
    """Load the CUDA library once; raise DeviceError if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(f"{LIB_PATH} is missing: build it with `python -m paper_1501_02946_b200._build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().patfft_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    """Map an ABI status code onto the reference's exception classes."""
    if rc == PATFFT_OK:
        return
    msg = last_error() or what
    if rc == PATFFT_ERR_PARAMETER:
        raise ParameterError(msg)
    if rc == PATFFT_ERR_DATA:
        raise DataValidationError(msg)
    if rc == PATFFT_ERR_UNSUPPORTED:
        raise DeviceError(f"unsupported on the GPU path: {msg}")
    raise DeviceError(msg)


def ptr(a) -> ctypes.c_void_p:
    """Raw pointer of a numpy array (host) -- must be C-contiguous."""
    return ctypes.c_void_p(a.ctypes.data)


def device_count() -> int:
    n = ctypes.c_int(0)
    rc = load().patfft_device_count(ctypes.byref(n))
    return n.value if rc == PATFFT_OK else 0

"""ctypes binding of the sm_100a C-ABI (include/shockhash_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``) into ``paper_2308_09561_b200/_lib``.
There is exactly one backend and no CPU fallback: if the library or a B200 is
missing, every compute call raises ``BackendUnavailableError``.
"""

import ctypes
import os
import threading

import numpy as np

from ..errors import (
    ConstructionFailureError,
    FormatError,
    HashCollisionError,
    InvalidParameterError,
    ShockHashError,
)

LIB_PATH = os.environ.get("SHK_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "_lib", "libshockhash_b200.so")

SHK_OK, SHK_EXHAUSTED, SHK_FORMAT, SHK_INVALID, SHK_UNSOLVABLE, SHK_DUPLICATE = range(6)
SHK_DEVICE = 1
SHK_BUILD_ASYNC = 8


class BackendUnavailableError(ShockHashError, RuntimeError):
    """The CUDA library or a usable B200 is missing (there is no CPU fallback)."""


class ShkPlans(ctypes.Structure):
    _fields_ = [
        ("nplans", ctypes.c_int64),
        ("plan_m", ctypes.c_void_p),
        ("plan_off", ctypes.c_void_p),
        ("sizes_base", ctypes.c_void_p),
        ("kind", ctypes.c_void_p),
        ("g", ctypes.c_void_p),
        ("fanout", ctypes.c_void_p),
        ("sizes_off", ctypes.c_void_p),
        ("subtree", ctypes.c_void_p),
        ("m_node", ctypes.c_void_p),
        ("sizes_flat", ctypes.c_void_p),
    ]


_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64

# name -> (restype, argtypes)
_SIGS = {
    "shk_last_error": (ctypes.c_char_p, []),
    "shk_version": (_I, []),
    "shk_device_count": (_I, [_P]),
    "shk_ctx_create": (_I, [_I, _P]),
    "shk_ctx_destroy": (_I, [_P]),
    "shk_ctx_sync": (_I, [_P]),
    "shk_ctx_stream": (_P, [_P]),
    "shk_ctx_set_stream": (_I, [_P, _P]),
    "shk_ctx_num_sms": (_I, [_P]),
    "shk_ctx_set_option": (_I, [_P, _I, _I64]),
    "shk_int_peak": (_I, [_P, _I, _I, _P, _P]),
    "shk_ipc_counter_alloc": (_I, [_P, _P, _P]),
    "shk_ipc_counter_open": (_I, [_P, _P, _P]),
    "shk_ipc_counter_close": (_I, [_P, _P, _I]),
    "shk_ipc_counter_reset": (_I, [_P, _P]),
    "shk_ctx_set_leaf_counter": (_I, [_P, _P]),
    "shk_dev_alloc": (_I, [_P, ctypes.c_size_t, _P]),
    "shk_dev_free": (_I, [_P, _P]),
    "shk_host_alloc": (_I, [_P, ctypes.c_size_t, _P]),
    "shk_host_free": (_I, [_P, _P]),
    "shk_memcpy": (_I, [_P, _P, _P, ctypes.c_size_t, _I]),
    "shk_memset": (_I, [_P, _P, _I, ctypes.c_size_t]),
    "shk_exclusive_scan": (_I, [_P, _P, _P, _I64]),
    "shk_timer_start": (_I, [_P]),
    "shk_timer_stop": (_I, [_P, _P]),
    "shk_launch_count": (_I64, [_P]),
    "shk_mix64": (_U64, [_U64]),
    "shk_seed_mixer": (_U64, [_U64, _U64]),
    "shk_remix": (_U64, [_U64, _U64, _U64, _U64]),
    "shk_hash_range": (_U64, [_U64, _U64]),
    "shk_leaf_pair": (None, [_U64, _U64, _U64, _I, _P, _P]),
    "shk_split_bit": (_I, [_U64, _U64, _U64]),
    "shk_leaf_cell": (_I, [_U64, _U64, _I64, _I, _I, _I64, _I]),
    "shk_leaf_search": (_I, [_P, _I, _I, _I, _P, _P, _P, _I64, _U64, _I, _P, _P, _P, _I]),
    "shk_orient": (_I, [_P, _P, _P, _P, _I64, _P, _P, _I]),
    "shk_split_search": (_I, [_P, _P, _P, _I64, _P, _I, _U64, _P, _P]),
    "shk_split_parts": (_I, [_P, _P, _P, _I64, _U64, _P, _I, _P]),
    "shk_ribbon_rows": (_I, [_P, _P, _P, _I64, _I64, _U64, _P, _P, _P, _I]),
    "shk_ribbon_solve": (_I, [_P, _P, _P, _P, _P, _I64, _I64, _P, _P, _I]),
    "shk_ribbon_query": (_I, [_P, _P, _P, _P, _I64, _P, _I64, _P, _I]),
    "shk_ribbon_build": (_I, [_P, _P, _P, _P, _I64, _I64, _I, _P, _P, _I]),
    "shk_rice_decode": (_I, [_P, _P, _I64, _I64, _I64, _P, _I64, _P, _P]),
    "shk_blake2b128": (_I, [_P, _P, _I64, _P, _I64, _U64, _P, _P, _I]),
    "shk_blake2b128_fixed": (_I, [_P, _P, _I, _I64, _U64, _P, _P, _I]),
    "shk_search_bruteforce": (_I, [_P, _P, _P, _I, _U64, _P, _P]),
    "shk_mc_filter_pass_count": (_I, [_P, _I, _I64, _U64, _P]),
    "shk_enumerate_outcomes": (_I, [_P, _I, _P, _P]),
    "shk_build_phase_ms": (_I, [_P, _P, _P]),
    "shk_build_level_ms": (_I, [_P, _P, _P, _I]),
    "shk_build_create": (_I, [_P, _P, _P, _I64, _I64, _I, _P, _P, _P]),
    "shk_build_duplicate": (_I, [_P, _P]),
    "shk_build_key_prefix": (_I, [_P, _P]),
    "shk_build_sorted_keys": (_I, [_P, _P, _P]),
    "shk_build_set_record_placements": (_I, [_P, _I]),
    "shk_build_placements": (_I, [_P, _P]),
    "shk_build_set_keep_sorted": (_I, [_P, _I]),
    "shk_build_choice_sorted": (_I, [_P, _I64, _I64, _P, _I]),
    "shk_build_dribbon_begin": (_I, [_P, _P, _I, _I64, _U64, _I64, _I64, _P, _P]),
    "shk_build_dribbon_map": (_I, [_P, _P]),
    "shk_build_dribbon_finish": (_I, [_P, _P, _P]),
    "shk_build_dribbon_exports": (_I, [_P, _P, _I64]),
    "shk_build_dribbon_begin_keys": (_I, [_P, _P, _P, _I64, _I64, _U64, _I64, _I64, _P, _P]),
    "shk_build_leaf_arrays": (_I, [_P, _P, _P]),
    "shk_route": (_I, [_P, _P, _P, _I64, _I, _U64, _U64, _P, _I, _P, _P, _P]),
    "shk_route_count": (_I, [_P, _P, _I64, _I, _U64, _U64, _P, _I, _P]),
    "shk_route_p2p": (_I, [_P, _P, _P, _I64, _I, _U64, _U64, _P, _I, _P, _P, _I64]),
    "shk_ipc_buffer_alloc": (_I, [_P, ctypes.c_size_t, _P, _P]),
    "shk_build_dribbon_import": (_I, [_P, _P, _I64, _P, _P]),
    "shk_build_dribbon_backsub": (_I, [_P, _P, _P, _P]),
    "shk_build_run": (_I, [_P, _P, _I, _I, _I, _I64, _I64, _U64, _P]),
    "shk_build_stream_size": (_I, [_P, _P, _P]),
    "shk_build_stream": (_I, [_P, _P, _P]),
    "shk_build_choice": (_I, [_P, _P]),
    "shk_build_ribbon": (_I, [_P, _P, _I, _I64, _I, _P, _P]),
    "shk_build_destroy": (_I, [_P]),
    "shk_qdesc_create": (_I, [_P, _I64, _I64, _I, _I64, _P, _P, _P, _I64, _I64, _P, _U64, _I64, _P, _I64, _P]),
    "shk_query": (_I, [_P, _P, _P, _I64, _P, _I, _I]),
    "shk_query_blob": (_I, [_P, _P, _I, _I64, _U64, _P, _I]),
    "shk_verify": (_I, [_P, _P, _P, _I64, _I, _P, _P]),
    "shk_qdesc_destroy": (_I, [_P]),
}

EXPORTED = sorted(_SIGS)

_lib = None
_lib_lock = threading.Lock()
_ctx = {}


def load_library(path: str = LIB_PATH):
    """Load the shared library (does not need a GPU)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise BackendUnavailableError(
                f"{path} is missing: run __graft_entry__.build() (nvcc, sm_100a). There is no CPU fallback."
            )
        lib = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error() -> str:
    lib = load_library()
    msg = lib.shk_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = ""):
    """Map a C-ABI status code onto the reference's exception hierarchy."""
    if rc == SHK_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == SHK_EXHAUSTED:
        raise ConstructionFailureError(msg)
    if rc == SHK_FORMAT:
        raise FormatError(msg)
    if rc == SHK_INVALID:
        raise InvalidParameterError(msg)
    if rc == SHK_UNSOLVABLE:
        raise ConstructionFailureError(msg)
    if rc == SHK_DUPLICATE:
        raise HashCollisionError(msg)
    raise BackendUnavailableError(f"CUDA failure ({rc}) {msg}")


def device_count() -> int:
    lib = load_library()
    n = ctypes.c_int(0)
    lib.shk_device_count(ctypes.byref(n))
    return n.value


def ctx(device: int = None):
    """Per-process, per-device context (stream + device memory pool)."""
    if device is None:
        device = int(os.environ.get("SHK_DEVICE", "0"))
    c = _ctx.get(device)
    if c is None:
        lib = load_library()
        h = ctypes.c_void_p()
        rc = lib.shk_ctx_create(device, ctypes.byref(h))
        if rc != SHK_OK:
            raise BackendUnavailableError(f"cannot create a CUDA context on device {device}: {last_error()}")
        c = h
        _ctx[device] = c
    return c


def ptr(a):
    """Data pointer of a contiguous numpy array (or None)."""
    if a is None:
        return None
    return a.ctypes.data


def u64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def i64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))

"""GPU-resident data for the hot path (benchmarks, zero-copy pipelines).

Device memory comes from the C-ABI context's caching pool; kernels run on the
context stream; ``timer`` brackets device work with CUDA events recorded on
that same stream (the stream the kernels are launched on).
"""

import ctypes

import numpy as np

from ._kernels import _lib
from ._kernels._lib import SHK_DEVICE, check, ctx


class DeviceBuffer:
    def __init__(self, nbytes: int):
        self.nbytes = int(nbytes)
        p = ctypes.c_void_p()
        check(_lib.load_library().shk_dev_alloc(ctx(), max(self.nbytes, 1), ctypes.byref(p)), "device alloc")
        self.ptr = p.value

    @classmethod
    def from_host(cls, a: np.ndarray) -> "DeviceBuffer":
        a = np.ascontiguousarray(a)
        b = cls(a.nbytes)
        b.upload(a)
        return b

    def upload(self, a: np.ndarray):
        a = np.ascontiguousarray(a)
        check(_lib.load_library().shk_memcpy(ctx(), self.ptr, a.ctypes.data, a.nbytes, 0), "H2D")

    def download(self, dtype, count) -> np.ndarray:
        out = np.empty(count, dtype=dtype)
        check(_lib.load_library().shk_memcpy(ctx(), out.ctypes.data, self.ptr, out.nbytes, 1), "D2H")
        return out

    def free(self):
        if self.ptr and _lib._lib is not None:
            _lib._lib.shk_dev_free(ctx(), self.ptr)
        self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class PinnedBuffer:
    """Page-locked host memory with a numpy view (``.array``)."""

    def __init__(self, nbytes: int, dtype=np.uint8):
        self.nbytes = int(nbytes)
        p = ctypes.c_void_p()
        check(_lib.load_library().shk_host_alloc(ctx(), max(self.nbytes, 1), ctypes.byref(p)), "host alloc")
        self.ptr = p.value
        buf = (ctypes.c_uint8 * max(self.nbytes, 1)).from_address(self.ptr)
        self.array = np.frombuffer(buf, dtype=np.uint8)[: self.nbytes].view(dtype)

    @classmethod
    def from_array(cls, a: np.ndarray) -> "PinnedBuffer":
        a = np.ascontiguousarray(a)
        b = cls(a.nbytes, a.dtype)
        b.array[...] = a.reshape(-1)
        return b

    def free(self):
        if self.ptr and _lib._lib is not None:
            self.array = None
            _lib._lib.shk_host_free(ctx(), self.ptr)
        self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def memset_device(ptr: int, value: int, nbytes: int):
    """Stream-ordered byte fill of device memory."""
    check(_lib.load_library().shk_memset(ctx(), ptr, int(value), int(nbytes)), "memset")


def exclusive_scan_device(d_in: "DeviceBuffer", d_out: "DeviceBuffer", n: int):
    """out[0..n] = exclusive prefix sum of n int64 values (out[n] = total), on the device."""
    check(_lib.load_library().shk_exclusive_scan(ctx(), d_in.ptr, d_out.ptr, int(n)), "scan")


def sync():
    check(_lib.load_library().shk_ctx_sync(ctx()), "sync")


class timer:
    """CUDA-event timing on the context stream: ``with timer() as t: ...; t.ms``."""

    def __enter__(self):
        check(_lib.load_library().shk_timer_start(ctx()))
        return self

    def __exit__(self, *exc):
        ms = ctypes.c_float(0)
        check(_lib.load_library().shk_timer_stop(ctx(), ctypes.byref(ms)))
        self.ms = float(ms.value)
        return False


OPT_EXACT_SPLIT_EVALS = 0
OPT_LEAF_TEAM_WARPS = 1
OPT_SCHEDULE = 2  # 0 persistent task queue (default), 1 one launch per tree level
OPT_LEAF_FIXED_TEAMS = 3  # 1: plain batched leaf search with fixed teams (no seed-block stealing)


def set_option(opt: int, value: int):
    """Context tuning/instrumentation option (include/shockhash_b200.h)."""
    check(_lib.load_library().shk_ctx_set_option(ctx(), int(opt), int(value)), "option")


INT_PEAK_KINDS = {0: "LOP3", 1: "IMAD", 2: "LOP3+IMAD 1:1", 3: "SHF+LOP3+IMAD 2:1:1"}
# analysis only (tools/int_peak.py): pipe cost of the hash's multiply forms
INT_PEAK_KINDS_EXTRA = {4: "IMAD.WIDE", 5: "IMAD.HI", 6: "IMAD.WIDE+LOP3 1:1", 7: "IMAD.HI+LOP3 1:1",
                        8: "IMAD(2^k)+LOP3 1:1"}


def int_peak(kind: int, iters: int = 4096):
    """(ms, int32 ops) of one timed launch of the integer-issue
    microbenchmark (csrc/shk_peak.cu; kinds in INT_PEAK_KINDS)."""
    import ctypes

    ms = ctypes.c_double()
    ops = ctypes.c_double()
    check(_lib.load_library().shk_int_peak(ctx(), int(kind), int(iters), ctypes.byref(ms), ctypes.byref(ops)),
          "int peak")
    return ms.value, ops.value


def launch_count() -> int:
    return int(_lib.load_library().shk_launch_count(ctx()))


def num_sms() -> int:
    return int(_lib.load_library().shk_ctx_num_sms(ctx()))


def blake2b_fixed_device(d_blob: DeviceBuffer, key_len: int, N: int, salt: int, d_hi: DeviceBuffer, d_lo: DeviceBuffer):
    check(_lib.load_library().shk_blake2b128_fixed(ctx(), d_blob.ptr, int(key_len), int(N), int(salt), d_hi.ptr,
                                                   d_lo.ptr, SHK_DEVICE), "blake2b")


SHK_BLOB_HOST = 2


def blake2b_fixed_from_host(blob: np.ndarray, key_len: int, N: int, salt: int, d_hi: DeviceBuffer,
                            d_lo: DeviceBuffer):
    """Host key blob (ideally a PinnedBuffer's array) -> device codes; the
    H2D copy is chunked and overlapped with the hashing."""
    blob = np.ascontiguousarray(blob, dtype=np.uint8)
    check(_lib.load_library().shk_blake2b128_fixed(ctx(), blob.ctypes.data, int(key_len), int(N), int(salt), d_hi.ptr,
                                                   d_lo.ptr, SHK_BLOB_HOST), "blake2b")


def blake2b_fixed_host(blob: np.ndarray, key_len: int, salt: int = 0):
    """Host buffers in, host codes out; H2D/D2H inside the call."""
    blob = np.ascontiguousarray(blob, dtype=np.uint8)
    N = len(blob) // key_len
    hi = np.empty(N, dtype=np.uint64)
    lo = np.empty(N, dtype=np.uint64)
    check(_lib.load_library().shk_blake2b128_fixed(ctx(), blob.ctypes.data, int(key_len), N, int(salt),
                                                   hi.ctypes.data, lo.ctypes.data, 0), "blake2b")
    return hi, lo

"""ctypes binding of libucores_cuda.so (include/ucores_cuda.h).

This is the "reference-side binding a maintainer would add" for Python
callers; bench.py and the tests drive the CUDA path through
it. There is no fallback: if the library or a sm_100 device is missing, every
compute call raises.
"""
from __future__ import annotations

import array
import ctypes as C
import os
from pathlib import Path
from typing import Sequence

from .errors import DeviceUnavailable, EmptyDataset, KernelPanic, LengthMismatch, PeerExchangeError

LIB_DIR = Path(__file__).resolve().parent / "_lib"
LIB_PATH = LIB_DIR / "libucores_cuda.so"

OK, ERR_CUDA, ERR_ARG, ERR_NODEV, ERR_LENGTH, ERR_EMPTY, ERR_NCCL, ERR_PEER = 0, -1, -2, -3, -4, -5, -6, -7
OP_SUM, OP_MAX = 0, 1
OPS = {"sum": OP_SUM, "max": OP_MAX}

vp, u64, i32, f32 = C.c_void_p, C.c_uint64, C.c_int, C.c_float
P = C.POINTER


class DeviceInfo(C.Structure):
    _fields_ = [("name", C.c_char * 128), ("ordinal", C.c_int), ("cc_major", C.c_int), ("cc_minor", C.c_int),
                ("sm_count", C.c_int), ("hbm_bytes", C.c_uint64), ("l2_bytes", C.c_uint64)]


# name -> (restype, argtypes)
SIGNATURES: dict[str, tuple] = {
    "ucg_last_error": (C.c_char_p, []),
    "ucg_abi_version": (i32, []),
    "ucg_device_count": (i32, [P(C.c_int)]),
    "ucg_device_info_get": (i32, [C.c_int, P(DeviceInfo)]),
    "ucg_set_device": (i32, [C.c_int]),
    "ucg_get_device": (i32, [C.POINTER(C.c_int)]),
    "ucg_malloc": (i32, [P(vp), u64]),
    "ucg_free": (i32, [vp]),
    "ucg_host_alloc": (i32, [P(vp), u64]),
    "ucg_host_free": (i32, [vp]),
    "ucg_host_register": (i32, [vp, u64]),
    "ucg_host_unregister": (i32, [vp]),
    "ucg_memcpy_h2d": (i32, [vp, vp, u64, vp]),
    "ucg_memcpy_d2h": (i32, [vp, vp, u64, vp]),
    "ucg_memcpy_d2d": (i32, [vp, vp, u64, vp]),
    "ucg_memcpy2d": (i32, [vp, u64, vp, u64, u64, u64, vp]),
    "ucg_memset": (i32, [vp, C.c_int, u64, vp]),
    "ucg_stream_create": (i32, [P(vp)]),
    "ucg_stream_destroy": (i32, [vp]),
    "ucg_stream_synchronize": (i32, [vp]),
    "ucg_event_create": (i32, [P(vp)]),
    "ucg_event_destroy": (i32, [vp]),
    "ucg_event_record": (i32, [vp, vp]),
    "ucg_event_synchronize": (i32, [vp]),
    "ucg_stream_wait_event": (i32, [vp, vp]),
    "ucg_event_elapsed_ms": (i32, [vp, vp, P(f32)]),
    "ucg_device_synchronize": (i32, []),
    "ucg_launch_count": (u64, []),
    "ucg_fill_uniform_f32": (i32, [vp, u64, u64, u64, vp]),
    "ucg_fill_bytes_u8": (i32, [vp, u64, u64, u64, vp]),
    "ucg_segtab_create": (i32, [P(u64), P(u64), u64, P(vp)]),
    "ucg_segtab_destroy": (i32, [vp]),
    "ucg_segtab_scratch_floats": (i32, [vp, P(u64)]),
    "ucg_map_affine_f32": (i32, [vp, vp, u64, f32, f32, vp]),
    "ucg_elementwise2_f32": (i32, [vp, vp, vp, u64, C.c_int, vp]),
    "ucg_elementwise2_i64": (i32, [vp, vp, vp, u64, vp]),
    "ucg_segment_reduce_f32": (i32, [vp, vp, C.c_int, vp, vp, vp]),
    "ucg_map_affine_segment_reduce_f32": (i32, [vp, vp, vp, f32, f32, C.c_int, vp, vp, vp]),
    "ucg_tree_reduce_f32": (i32, [vp, u64, C.c_int, vp, vp]),
    "ucg_xchg_create": (i32, [C.c_int, C.c_int, u64, u64, u64, P(vp)]),
    "ucg_xchg_handle_bytes": (u64, []),
    "ucg_xchg_export": (i32, [vp, vp]),
    "ucg_xchg_open": (i32, [vp, vp]),
    "ucg_xchg_error": (i32, [vp, P(C.c_int)]),
    "ucg_xchg_poll": (i32, [vp, P(C.c_int)]),
    "ucg_xchg_reset": (i32, [vp]),
    "ucg_xchg_destroy": (i32, [vp]),
    "ucg_segment_reduce_cl_f32": (i32, [vp, vp, vp, f32, f32, C.c_int, vp, vp, vp, vp, vp]),
    "ucg_reduce_cl_f32": (i32, [vp, u64, u64, P(u64), u64, C.c_int, vp, vp]),
    "ucg_reduce_cl_i64": (i32, [vp, u64, u64, P(u64), u64, vp, vp]),
    "ucg_pi_hits": (i32, [P(u64), P(u64), u64, vp, vp]),
    "ucg_pi_hits_total": (i32, [P(u64), P(u64), u64, vp, vp, vp]),
    "ucg_pi_hits_total_xchg": (i32, [P(u64), P(u64), u64, vp, vp, vp, vp]),
    "ucg_reduce_cl_xchg_f32": (i32, [vp, u64, C.c_int, vp, vp, vp]),
    "ucg_pi_flags": (i32, [u64, u64, vp, vp]),
    "ucg_sobel_band_u8": (i32, [vp, vp, u64, u64, vp]),
    "ucg_sobel_bands_u8": (i32, [vp, P(u64), vp, P(u64), P(u64), u64, u64, vp]),
    "ucg_gemm_tf32": (i32, [vp, vp, vp, u64, vp]),
    "ucg_gemm_f32": (i32, [vp, vp, vp, u64, vp]),
    "ucg_word_start_flags": (i32, [vp, u64, vp, vp]),
}

_lib: C.CDLL | None = None


def load() -> C.CDLL:
    """Load the in-tree library (raises DeviceUnavailable if it was never built)."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("UCORES_CUDA_LIB", LIB_PATH))
    if not path.exists():
        raise DeviceUnavailable(f"{path} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    lib = C.CDLL(str(path))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    return load().ucg_last_error().decode(errors="replace")


def check(rc: int, what: str = "run") -> None:
    """Map a status code onto the reference's exceptions."""
    if rc == OK:
        return
    msg = last_error()
    if rc == ERR_NODEV:
        raise DeviceUnavailable(msg)
    if rc == ERR_LENGTH:
        raise LengthMismatch(msg)
    if rc == ERR_EMPTY:
        raise EmptyDataset(msg)
    if rc == ERR_PEER:
        raise PeerExchangeError(what, msg)
    raise KernelPanic(what, msg)


def call(name: str, *args, phase: str = "run") -> None:
    check(getattr(load(), name)(*args), phase)


def u64_array(vals: Sequence[int]) -> C.Array:
    """A C uint64 array of `vals` (negative or > 2^64-1 values raise OverflowError)."""
    if not len(vals):
        return (C.c_uint64 * 1)()
    return (C.c_uint64 * len(vals)).from_buffer_copy(array.array("Q", vals))


def ptr(x) -> int | None:
    """Device pointer of a torch tensor / int / None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()


def stream_handle(stream=None) -> int | None:
    """cudaStream_t of a torch stream (current stream by default)."""
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def device_count() -> int:
    n = C.c_int(0)
    call("ucg_device_count", C.byref(n))
    return n.value


def device_info(ordinal: int = 0) -> DeviceInfo:
    info = DeviceInfo()
    call("ucg_device_info_get", ordinal, C.byref(info))
    return info


def launch_count() -> int:
    return int(load().ucg_launch_count())


class SegTab:
    """Owned handle of a device segment table (one Dataset layout)."""

    def __init__(self, begins: Sequence[int], lens: Sequence[int]):
        self.nseg = len(begins)
        # the furthest float any segment touches: x / y must cover it
        self.max_end = max((int(b) + int(n) for b, n in zip(begins, lens)), default=0)
        h = vp()
        call("ucg_segtab_create", u64_array(begins), u64_array(lens), self.nseg, C.byref(h), phase="map_parameters")
        self.handle = h.value
        n = u64()
        call("ucg_segtab_scratch_floats", self.handle, C.byref(n))
        self.scratch_floats = int(n.value)

    def close(self) -> None:
        if self.handle:
            load().ucg_segtab_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

"""ctypes binding of libucores_engine.so (include/ucores_engine.h): the
unmodified reference ucores::Engine driven through the B200 drop-in drivers
(GpuClusterDriver, seam A; GpuWorkerRuntime/CudaExecutor, seam B)."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from . import capi
from .errors import ArityMismatch, EmptyDataset, Error, JobFailed, UnknownKernel

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libucores_engine.so"
MODE = {"batched": 0, "per_task": 1, "device": 2}
_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is None:
        capi.load()  # resolves libucores_cuda.so first
        if not LIB_PATH.exists():
            raise capi.DeviceUnavailable(f"{LIB_PATH} missing (built where the reference headers exist)")
        L = C.CDLL(str(LIB_PATH))
        L.ucd_last_error.restype = C.c_char_p
        L.ucd_pipeline_f32.restype = C.c_int
        L.ucd_pipeline_f32.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.c_uint64, C.c_float, C.c_float, C.c_int,
                                       C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_float),
                                       C.POINTER(C.c_double)]
        L.ucd_pipeline_breakdown_f32.restype = C.c_int
        L.ucd_pipeline_breakdown_f32.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.c_uint64, C.c_float, C.c_float,
                                                 C.c_int, C.c_int, C.c_void_p]
        L.ucd_literal_f32.restype = C.c_int
        L.ucd_literal_f32.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_float, C.c_float, C.c_int, C.c_int,
                                      C.c_int, C.POINTER(C.c_float), C.POINTER(C.c_double)]
        L.ucd_pi.restype = C.c_int
        L.ucd_pi.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_double)]
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = load().ucd_last_error().decode(errors="replace")
    raise {-10: JobFailed, -11: EmptyDataset, -12: ArityMismatch, -13: UnknownKernel}.get(rc, Error)(msg)


def pipeline_f32(x: np.ndarray, part_lens, a: float = 2.0, b: float = 1.0, op: str = "sum", gpus: int = -1,
                 mode: str = "batched", want_y: bool = True):
    """y, partials, result, seconds of map_cl(axpb)->map_cl_partition(p<op>)->reduce_cl(<op>2)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    lens = capi.u64_array(part_lens)
    y = np.empty_like(x) if want_y else None
    partials = np.empty(len(part_lens), np.float32)
    res, sec = C.c_float(0), C.c_double(0)
    _check(load().ucd_pipeline_f32(x.ctypes.data, lens, len(part_lens), a, b, capi.OPS[op], gpus, MODE[mode],
                                   y.ctypes.data if want_y else None, partials.ctypes.data, C.byref(res),
                                   C.byref(sec)))
    return y, partials, np.float32(res.value), sec.value


def pipeline_breakdown_f32(x: np.ndarray, part_lens, a: float = 2.0, b: float = 1.0, op: str = "sum",
                           gpus: int = -1) -> dict:
    """Seconds of each reference Engine call of the C2 chain through seam A,
    split into the driver's run_wave time and the Engine's own work."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.zeros(8, np.float64)
    _check(load().ucd_pipeline_breakdown_f32(x.ctypes.data, capi.u64_array(part_lens), len(part_lens), a, b,
                                             capi.OPS[op], gpus, out.ctypes.data))
    keys = ["map_cl_s", "map_cl_wave_s", "map_cl_partition_s", "map_cl_partition_wave_s", "reduce_cl_s",
            "reduce_cl_wave_s", "total_s"]
    d = {k: float(v) for k, v in zip(keys, out[:7])}
    d["engine_own_s"] = d["total_s"] - d["map_cl_wave_s"] - d["map_cl_partition_wave_s"] - d["reduce_cl_wave_s"]
    d["result_bits"] = "%08x" % int(out[7])
    return d


def literal_f32(x: np.ndarray, parts: int, a: float = 2.0, b: float = 1.0, op: str = "sum", gpus: int = -1,
                mode: str = "device"):
    """C1 literal form: one-float elements; (result, seconds) of the same chain."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    res, sec = C.c_float(0), C.c_double(0)
    _check(load().ucd_literal_f32(x.ctypes.data, x.size, parts, a, b, capi.OPS[op], gpus, MODE[mode], C.byref(res),
                                  C.byref(sec)))
    return np.float32(res.value), sec.value


def pi(samples: int, tasks: int, seed: int, gpus: int = -1):
    h, sec = C.c_int64(0), C.c_double(0)
    _check(load().ucd_pi(samples, tasks, seed, gpus, C.byref(h), C.byref(sec)))
    return int(h.value), sec.value

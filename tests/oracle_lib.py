"""ctypes access to the C oracle (oracle/_build/liboracle.so) — test checker only."""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE_SO = ROOT / "oracle" / "_build" / "liboracle.so"
REF_HARNESS = ROOT / "oracle" / "_ref" / "ref_harness"

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not ORACLE_SO.exists():
            subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "_build/liboracle.so"], check=True)
        L = C.CDLL(str(ORACLE_SO))
        vp, u64, f32 = C.c_void_p, C.c_uint64, C.c_float
        sig = {
            "orc_mix64": (u64, [u64]),
            "orc_stream_u64": (u64, [u64, u64]),
            "orc_fill_uniform_f32": (None, [u64, u64, u64, vp]),
            "orc_fill_vectoradd": (None, [u64, u64, vp]),
            "orc_fnv64": (u64, [vp, u64]),
            "orc_partition_sizes": (C.c_int, [u64, u64, vp]),
            "orc_map_affine_f32": (None, [vp, u64, f32, f32, vp]),
            "orc_tree_reduce_f32": (f32, [vp, u64, C.c_int]),
            "orc_tree_reduce_i64": (C.c_int64, [vp, u64]),
            "orc_reduce_cl_f32": (C.c_int, [vp, u64, vp, u64, C.c_int, vp]),
            "orc_reduce_cl_i64": (C.c_int, [vp, u64, vp, u64, vp]),
            "orc_pi_hit": (C.c_int, [u64, u64]),
            "orc_pi_hits": (u64, [u64, u64]),
            "orc_sobel_band_u8": (None, [vp, u64, u64, vp]),
            "orc_matmul_f32": (None, [vp, vp, u64, vp]),
            "orc_matmul_entry_f64": (C.c_double, [vp, vp, u64, u64, u64]),
            "orc_word_start_flags": (None, [vp, u64, vp]),
            "orc_chunk_offsets": (u64, [vp, u64, u64, vp, u64]),
        }
        for k, (r, a) in sig.items():
            f = getattr(L, k)
            f.restype, f.argtypes = r, a
        _lib = L
    return _lib


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


OP = {"sum": 0, "max": 1}


def fill_uniform(seed: int, n: int, first: int = 0) -> np.ndarray:
    out = np.empty(n, dtype=np.float32)
    lib().orc_fill_uniform_f32(seed, first, n, _p(out))
    return out


def fill_vectoradd(k: int, length: int) -> np.ndarray:
    out = np.empty(length, dtype=np.float32)
    lib().orc_fill_vectoradd(k, length, _p(out))
    return out


def fnv64(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    return "%016x" % lib().orc_fnv64(_p(a), a.nbytes)


def partition_sizes(n: int, p: int) -> list[int]:
    out = np.zeros(max(p, 1), dtype=np.uint64)
    if lib().orc_partition_sizes(n, p, _p(out)) != 0:
        raise ValueError("InvalidPartitionCount")
    return [int(v) for v in out[:p]]


def map_affine(x: np.ndarray, a: float, b: float) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    y = np.empty_like(x)
    lib().orc_map_affine_f32(_p(x), x.size, a, b, _p(y))
    return y


def tree_reduce(x: np.ndarray, op: str = "sum") -> np.float32:
    x = np.ascontiguousarray(x, dtype=np.float32)
    return np.float32(lib().orc_tree_reduce_f32(_p(x), x.size, OP[op]))


def tree_reduce_i64(x: np.ndarray) -> int:
    x = np.ascontiguousarray(x, dtype=np.int64)
    return int(lib().orc_tree_reduce_i64(_p(x), x.size))


def reduce_cl(elems: np.ndarray, part_counts: list[int], op: str = "sum") -> np.ndarray:
    """elems: [count, len] array in collect() order."""
    pc = np.asarray(part_counts, dtype=np.uint64)
    if elems.dtype == np.int64:
        e = np.ascontiguousarray(elems)
        out = np.empty(e.shape[1], dtype=np.int64)
        rc = lib().orc_reduce_cl_i64(_p(e), e.shape[1], _p(pc), pc.size, _p(out))
    else:
        e = np.ascontiguousarray(elems, dtype=np.float32)
        out = np.empty(e.shape[1], dtype=np.float32)
        rc = lib().orc_reduce_cl_f32(_p(e), e.shape[1], _p(pc), pc.size, OP[op], _p(out))
    if rc != 0:
        raise ValueError("EmptyDataset")
    return out


def pi_hits(seed: int, samples: int) -> int:
    return int(lib().orc_pi_hits(seed, samples))


def sobel_band(band: np.ndarray, rows_out: int, width: int) -> np.ndarray:
    band = np.ascontiguousarray(band, dtype=np.uint8)
    out = np.empty(rows_out * width, dtype=np.uint8)
    lib().orc_sobel_band_u8(_p(band), rows_out, width, _p(out))
    return out


def matmul(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    n = A.shape[0]
    A = np.ascontiguousarray(A, dtype=np.float32)
    B = np.ascontiguousarray(B, dtype=np.float32)
    Cm = np.empty((n, n), dtype=np.float32)
    lib().orc_matmul_f32(_p(A), _p(B), n, _p(Cm))
    return Cm


def matmul_entry_f64(A: np.ndarray, B: np.ndarray, i: int, j: int) -> float:
    return float(lib().orc_matmul_entry_f64(_p(A), _p(B), A.shape[0], i, j))


def stream_u64(seed: int, i: int) -> int:
    return int(lib().orc_stream_u64(seed, i))


def mix64(z: int) -> int:
    return int(lib().orc_mix64(z & 0xFFFFFFFFFFFFFFFF))


def sobel_image(H: int, W: int, seed: int) -> np.ndarray:
    """Counter-hash image: pixel i = mix64(seed + (i+1)*GAMMA) >> 56 (row-major)."""
    g = 0x9E3779B97F4A7C15
    i = np.arange(H * W, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (i + np.uint64(1)) * np.uint64(g)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(56)).astype(np.uint8).reshape(H, W)


def sobel_bands(img: np.ndarray, rows: int) -> list[np.ndarray]:
    """Row bands of `rows` output rows with one halo row above/below (zero outside)."""
    H, W = img.shape
    bands = []
    for r0 in range(0, H, rows):
        rr = min(rows, H - r0)
        b = np.zeros((rr + 2, W), dtype=np.uint8)
        for k in range(rr + 2):
            src = r0 + k - 1
            if 0 <= src < H:
                b[k] = img[src]
        bands.append(b)
    return bands


def word_start_flags(data: bytes) -> np.ndarray:
    b = np.frombuffer(data, dtype=np.uint8).copy()
    out = np.empty(b.size, dtype=np.uint8)
    lib().orc_word_start_flags(_p(b), b.size, _p(out))
    return out


def chunk_offsets(data: bytes, target: int) -> list[tuple[int, int]]:
    b = np.frombuffer(data, dtype=np.uint8).copy()
    cap = len(data) // max(1, target) + 2
    pairs = np.zeros(2 * cap, dtype=np.uint64)
    k = int(lib().orc_chunk_offsets(_p(b), b.size, target, _p(pairs), cap))
    return [(int(pairs[2 * i]), int(pairs[2 * i + 1])) for i in range(k)]


def corpus(seed: int, words: int) -> bytes:
    """Synthetic text shared with oracle/ref_harness.cpp make_corpus."""
    dl = b" \t\n\r"
    out = bytearray()
    for i in range(words):
        z = mix64(seed + i)
        out += b"w" + str(z % 97).encode()
        out += bytes([dl[(z >> 32) & 3]]) * (1 + ((z >> 40) & 1))
    return bytes(out)


def word_table(chunk: bytes, flags=None) -> list[tuple[bytes, int]]:
    """KeyCountTable of one chunk, keys in first-occurrence order (from flags
    when given, else by direct tokenisation) — small inputs only."""
    delim = set(b" \t\n\r")
    order, counts = [], {}
    n = len(chunk)
    starts = [i for i in range(n) if flags[i]] if flags is not None else None
    if starts is None:
        starts, i = [], 0
        while i < n:
            while i < n and chunk[i] in delim:
                i += 1
            if i < n:
                starts.append(i)
            while i < n and chunk[i] not in delim:
                i += 1
    for s in starts:
        e = s
        while e < n and chunk[e] not in delim:
            e += 1
        k = chunk[s:e]
        if k not in counts:
            order.append(k)
            counts[k] = 0
        counts[k] += 1
    return [(k, counts[k]) for k in order]


def f32_bits(v) -> str:
    return "%08x" % int(np.asarray(v, dtype=np.float32).view(np.uint32))

"""Typed wrappers over the C-ABI for torch-owned device memory.

Each wrapper names the reference operation it implements. Tensors must live on
the current CUDA device; work is enqueued on the current torch stream (or the
`stream` given), so CUDA events recorded by torch bracket it correctly.
"""
from __future__ import annotations

from typing import Sequence

import ctypes as C

from . import capi
from .capi import call, ptr, stream_handle, u64_array


def _require_cuda(*ts) -> None:
    """Every tensor handed to the C-ABI is a contiguous buffer on the current
    CUDA device (the kernels index raw pointers and run on that device)."""
    cur = None
    for t in ts:
        if t is None:
            continue
        if not t.is_cuda:
            raise capi.DeviceUnavailable("tensor is not on a CUDA device (no CPU fallback)")
        if not t.is_contiguous():
            raise ValueError("tensor must be contiguous (the C-ABI takes raw pointers)")
        if cur is None:
            import torch

            cur = torch.cuda.current_device()
        if t.device.index != cur:
            raise ValueError(f"tensor is on cuda:{t.device.index} but the current device is cuda:{cur}")


def _dtype(t, want, name: str) -> None:
    if t is not None and t.dtype != want:
        raise TypeError(f"{name} must be {want}, got {t.dtype}")


def _f32(*named) -> None:
    import torch

    for name, t in named:
        _dtype(t, torch.float32, name)


def _at_least(t, n: int, name: str) -> None:
    if t is not None and t.numel() < n:
        raise ValueError(f"{name} holds {t.numel()} elements, needs >= {n}")


def _check_segments(segtab: capi.SegTab, x, y, scratch, partials) -> None:
    """Every buffer a segment-table launch indexes covers the extents the
    table implies: x / y its furthest segment end, scratch its item roots,
    partials one value per segment."""
    _f32(("x", x), ("y", y), ("scratch", scratch), ("partials", partials))
    _at_least(x, segtab.max_end, "x")
    _at_least(y, segtab.max_end, "y")
    _at_least(scratch, segtab.scratch_floats, "scratch")
    _at_least(partials, segtab.nseg, "partials")


def fill_uniform_(out, seed: int, first: int = 0, stream=None):
    """Synthetic U[0,1) input: out[i] = (mix64(seed + (first+i+1)*GAMMA) >> 40) * 2^-24."""
    _require_cuda(out)
    call("ucg_fill_uniform_f32", ptr(out), out.numel(), seed, first, stream_handle(stream))
    return out


def fill_bytes_(out, seed: int, first: int = 0, stream=None):
    _require_cuda(out)
    call("ucg_fill_bytes_u8", ptr(out), out.numel(), seed, first, stream_handle(stream))
    return out


def map_affine(x, y, a: float, b: float, n: int | None = None, stream=None):
    """axpb mapCL body (engine.hpp:54-85): y = fl(fl(a*x)+b)."""
    _require_cuda(x, y)
    import torch

    _dtype(x, torch.float32, "x")
    _dtype(y, torch.float32, "y")
    if (x.numel() if n is None else n) > min(x.numel(), y.numel()):
        raise ValueError("n exceeds the buffers")
    call("ucg_map_affine_f32", ptr(x), ptr(y), x.numel() if n is None else n, a, b, stream_handle(stream))
    return y


def elementwise2(a, b, c, op: str = "sum", stream=None):
    """Fig-3 vectoradd body c = a (op) b (sum2 / max2 / isum2)."""
    _require_cuda(a, b, c)
    if a.numel() != b.numel():
        raise capi.LengthMismatch("vector lengths differ")
    import torch

    if not (a.dtype == b.dtype == c.dtype) or a.dtype not in (torch.float32, torch.int64):
        raise TypeError("a, b, c must all be float32 or all int64")
    _at_least(c, a.numel(), "c")

    if a.dtype == torch.int64:
        call("ucg_elementwise2_i64", ptr(a), ptr(b), ptr(c), a.numel(), stream_handle(stream))
    else:
        call("ucg_elementwise2_f32", ptr(a), ptr(b), ptr(c), a.numel(), capi.OPS[op], stream_handle(stream))
    return c


def segment_reduce(x, segtab: capi.SegTab, op: str, scratch, out, stream=None):
    """mapCLPartition psum/pmax over every segment (engine.hpp:89-114)."""
    _require_cuda(x, scratch, out)
    _check_segments(segtab, x, None, scratch, out)
    call("ucg_segment_reduce_f32", ptr(x), segtab.handle, capi.OPS[op], ptr(scratch), ptr(out),
         stream_handle(stream))
    return out


def map_affine_segment_reduce(x, y, segtab: capi.SegTab, a: float, b: float, op: str, scratch, out, stream=None):
    """Fused mapCL(axpb) -> mapCLPartition(psum|pmax): y written, partials reduced."""
    _require_cuda(x, y, scratch, out)
    _check_segments(segtab, x, y, scratch, out)
    call("ucg_map_affine_segment_reduce_f32", ptr(x), ptr(y), segtab.handle, a, b, capi.OPS[op], ptr(scratch),
         ptr(out), stream_handle(stream))
    return out


def segment_reduce_cl(x, y, segtab: capi.SegTab, a: float, b: float, op: str, scratch, partials, xchg, result,
                      stream=None):
    """map_cl(axpb) (when y is given) -> map_cl_partition(p<op>) -> reduce_cl(<op>2) in one launch;
    xchg (a ucg_xchg handle) makes the last stage a fused cross-GPU exchange."""
    _require_cuda(x, y, scratch, partials, result)
    _check_segments(segtab, x, y, scratch, partials)
    _f32(("result", result))
    _at_least(result, 1, "result")
    call("ucg_segment_reduce_cl_f32", ptr(x), ptr(y), segtab.handle, a, b, capi.OPS[op], ptr(scratch), ptr(partials),
         xchg, ptr(result), stream_handle(stream))
    return result


def tree_reduce(x, n: int, op: str, out, stream=None):
    """reduceCL stage 2 over n one-float partials (engine.hpp:172-190)."""
    _require_cuda(x, out)
    _f32(("x", x), ("out", out))
    _at_least(x, n, "x")
    _at_least(out, 1, "out")
    call("ucg_tree_reduce_f32", ptr(x), n, capi.OPS[op], ptr(out), stream_handle(stream))
    return out


def reduce_cl_vectors(elem_ptrs, count: int, length: int, part_counts: Sequence[int], op: str, out, dtype="f32",
                      stream=None):
    """Full reduceCL (stage 1 folds + stage 2 tree) over vector elements.

    elem_ptrs: int64 CUDA tensor holding the device addresses of the elements.
    """
    _require_cuda(elem_ptrs, out)
    import torch

    _dtype(elem_ptrs, torch.int64, "elem_ptrs")
    _dtype(out, torch.int64 if dtype == "i64" else torch.float32, "out")
    _at_least(elem_ptrs, count, "elem_ptrs")
    _at_least(out, length, "out")
    if sum(part_counts) != count:
        raise ValueError("part_counts do not sum to count")
    pc = u64_array(part_counts)
    if dtype == "i64":
        call("ucg_reduce_cl_i64", ptr(elem_ptrs), count, length, pc, len(part_counts), ptr(out),
             stream_handle(stream))
    else:
        call("ucg_reduce_cl_f32", ptr(elem_ptrs), count, length, pc, len(part_counts), capi.OPS[op], ptr(out),
             stream_handle(stream))
    return out


def pi_hits(seeds: Sequence[int], samples: Sequence[int], hits_out, stream=None, total_out=None, xchg=None):
    """Monte-Carlo pi mapCL over tasks {seed, samples}; with
    total_out, also the reduce_cl(isum2) of the task hits, in the same launch;
    with xchg (an opened exchange context, pipeline.open_exchange with 2 slots
    per rank), total_out is the sum over all ranks, exchanged over NVLink by
    the same kernel."""
    _require_cuda(hits_out)
    import torch

    if len(seeds) != len(samples):
        raise ValueError("one sample count per task seed")
    _dtype(hits_out, torch.int64, "hits_out")
    _dtype(total_out, torch.int64, "total_out")
    _at_least(hits_out, len(seeds), "hits_out")
    _at_least(total_out, 1, "total_out")
    if xchg is not None:
        _require_cuda(total_out)
        call("ucg_pi_hits_total_xchg", u64_array(seeds), u64_array(samples), len(seeds), ptr(hits_out),
             ptr(total_out), xchg, stream_handle(stream))
    elif total_out is None:
        call("ucg_pi_hits", u64_array(seeds), u64_array(samples), len(seeds), ptr(hits_out), stream_handle(stream))
    else:
        _require_cuda(total_out)
        call("ucg_pi_hits_total", u64_array(seeds), u64_array(samples), len(seeds), ptr(hits_out), ptr(total_out),
             stream_handle(stream))
    return hits_out


def sobel_bands(inp, in_off: Sequence[int], out, out_off: Sequence[int], rows: Sequence[int], width: int,
                stream=None):
    """mapCLPartition sobel over row bands (one launch for all bands)."""
    _require_cuda(inp, out)
    import torch

    _dtype(inp, torch.uint8, "inp")
    _dtype(out, torch.uint8, "out")
    if not (len(in_off) == len(out_off) == len(rows)):
        raise ValueError("one input offset, output offset and row count per band")
    if rows:  # the last band ends furthest when bands are laid out in order (the common case: check it first)
        in_end = in_off[-1] + (rows[-1] + 2) * width
        out_end = out_off[-1] + rows[-1] * width
        if in_end > inp.numel() or out_end > out.numel() or any(
                b < a for a, b in zip(in_off, in_off[1:])) or any(b < a for a, b in zip(out_off, out_off[1:])):
            _at_least(inp, max(o + (r + 2) * width for o, r in zip(in_off, rows)), "inp")
            _at_least(out, max(o + r * width for o, r in zip(out_off, rows)), "out")
    call("ucg_sobel_bands_u8", ptr(inp), u64_array(in_off), ptr(out), u64_array(out_off), u64_array(rows),
         len(rows), width, stream_handle(stream))
    return out


def word_start_flags(data, flags, stream=None):
    """wordcount run() over one chunk: 1 at every byte that starts a word."""
    _require_cuda(data, flags)
    import torch

    _dtype(data, torch.uint8, "data")
    _dtype(flags, torch.uint8, "flags")
    _at_least(flags, data.numel(), "flags")
    call("ucg_word_start_flags", ptr(data), data.numel(), ptr(flags), stream_handle(stream))
    return flags


def _check_gemm(A, B, Cm, n: int) -> None:
    _f32(("A", A), ("B", B), ("C", Cm))
    for name, t in (("A", A), ("B", B), ("C", Cm)):
        _at_least(t, n * n, name)


def gemm_tf32(A, B, Cm, n: int, stream=None):
    _require_cuda(A, B, Cm)
    _check_gemm(A, B, Cm, n)
    call("ucg_gemm_tf32", ptr(A), ptr(B), ptr(Cm), n, stream_handle(stream))
    return Cm


def gemm_f32(A, B, Cm, n: int, stream=None):
    """fp32-faithful C = A @ B on the tensor cores (3xTF32 split, ucg_gemm_f32)."""
    _require_cuda(A, B, Cm)
    _check_gemm(A, B, Cm, n)
    call("ucg_gemm_f32", ptr(A), ptr(B), ptr(Cm), n, stream_handle(stream))
    return Cm

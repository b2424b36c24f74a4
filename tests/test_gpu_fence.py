"""Electric-fence tests: every kernel family run on buffers that end (or start)
exactly at the edge of mapped device memory, with unmapped virtual address
space on the other side (CUDA VMM: cuMemAddressReserve + cuMemMap of only the
middle). A single out-of-bounds load or store in any kernel faults the
context (illegal address) instead of reading a neighbour's bytes silently;
the results are also checked against the oracle.

compute-sanitizer is closed on the GPU pool this project runs on, so these
fences (global-memory bounds, loads and stores) plus the ragged / empty /
special-value parity tests are the substitute. They do not cover
shared-memory races (racecheck) — the shared-memory protocols are covered by
bit-exact results over many shapes and repeated graph replays.
"""
import ctypes as C

import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _drv():
    from cuda.bindings import driver as d

    return d


def _ok(r):
    err = r[0] if isinstance(r, tuple) else r
    d = _drv()
    assert err == d.CUresult.CUDA_SUCCESS, err
    return r[1] if isinstance(r, tuple) and len(r) == 2 else r


class Fenced:
    """`nbytes` of device memory placed against an unmapped guard page:
    where="end": the last byte is followed by unmapped VA; "start": the first
    byte is preceded by unmapped VA."""

    def __init__(self, nbytes: int, where: str = "end"):
        d = _drv()
        torch.cuda.init()
        torch.empty(1, device="cuda")  # primary context current on this thread
        dev = torch.cuda.current_device()
        prop = d.CUmemAllocationProp()
        prop.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        prop.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        prop.location.id = dev
        gran = int(_ok(d.cuMemGetAllocationGranularity(
            prop, d.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_MINIMUM)))
        self.size = max(gran, (nbytes + gran - 1) // gran * gran)
        self.va = int(_ok(d.cuMemAddressReserve(self.size + 2 * gran, 0, 0, 0)))
        self.gran = gran
        self.handle = _ok(d.cuMemCreate(self.size, prop, 0))
        _ok(d.cuMemMap(self.va + gran, self.size, 0, self.handle, 0))
        acc = d.CUmemAccessDesc()
        acc.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = dev
        acc.flags = d.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        _ok(d.cuMemSetAccess(self.va + gran, self.size, [acc], 1))
        base = self.va + gran
        self.ptr = base + self.size - nbytes if where == "end" else base
        self.nbytes = nbytes

    def upload(self, a: np.ndarray) -> None:
        assert a.nbytes <= self.nbytes
        _ok(_drv().cuMemcpyHtoD(self.ptr, a.ctypes.data, a.nbytes))

    def download(self, dtype, count: int) -> np.ndarray:
        out = np.empty(count, dtype=dtype)
        if out.nbytes:
            _ok(_drv().cuMemcpyDtoH(out.ctypes.data, self.ptr, out.nbytes))
        return out

    def fill(self, byte: int) -> None:
        _ok(_drv().cuMemsetD8(self.ptr, byte, self.nbytes))

    def close(self) -> None:
        d = _drv()
        torch.cuda.synchronize()
        _ok(d.cuMemUnmap(self.va + self.gran, self.size))
        _ok(d.cuMemRelease(self.handle))
        _ok(d.cuMemAddressFree(self.va, self.size + 2 * self.gran))


def _sync_ok():
    torch.cuda.synchronize()  # an out-of-bounds access surfaces here as an illegal-address error


def _call(name, *args):
    from paper_1505_01120_b200 import capi

    capi.call(name, *args)


@pytest.mark.parametrize("where", ["end", "start"])
@pytest.mark.parametrize("n", [4, 1000, (1 << 20) + 12, 4096 * 148 * 17 + 4])
def test_fence_map_affine(cuda, n, where):
    x = O.fill_uniform(3, n)
    fx, fy = Fenced(4 * n, where), Fenced(4 * n, where)
    fx.upload(x)
    _call("ucg_map_affine_f32", fx.ptr, fy.ptr, n, 2.0, 1.0, None)
    _sync_ok()
    assert np.array_equal(fy.download(np.float32, n).view(np.uint32), O.map_affine(x, 2.0, 1.0).view(np.uint32))
    fx.close(), fy.close()


@pytest.mark.parametrize("where", ["end", "start"])
@pytest.mark.parametrize("lens", [[5], [100003, 65536, 1, 40000], [4096 * 3 + 7] * 9, [1 << 18] * 4,
                                  [(1 << 22) + 5, 17, (1 << 21)]])
@pytest.mark.parametrize("op", ["sum", "max"])
def test_fence_fused_segment_reduce_cl(cuda, lens, op, where):
    """k_segment_pass1 (claimed items, fused map, ticketed finisher tail and
    stage 2) with x, y, scratch, partials and result all fenced."""
    from paper_1505_01120_b200 import capi
    from paper_1505_01120_b200.pipeline import Layout

    lay = Layout.of(lens)
    total = lay.begins[-1] + lens[-1]  # the buffer ends with the last segment: no slack to hide over-reads
    tab = capi.SegTab(lay.begins, lens)
    fx, fy = Fenced(4 * ((total + 3) // 4 * 4), where), Fenced(4 * ((total + 3) // 4 * 4), where)
    fs = Fenced(4 * tab.scratch_floats, where)
    fp, fr = Fenced(4 * len(lens), where), Fenced(4, where)
    x = np.zeros((total + 3) // 4 * 4, np.float32)
    for k, n in enumerate(lens):
        x[lay.begins[k]:lay.begins[k] + n] = O.fill_uniform(1000 + k, n)
    fx.upload(x)
    for _ in range(2):  # the counters reset by the tail: a second launch is exact too
        _call("ucg_segment_reduce_cl_f32", fx.ptr, fy.ptr, tab.handle, 2.0, 1.0, capi.OPS[op], fs.ptr, fp.ptr, None,
              fr.ptr, None)
        _sync_ok()
    y = fy.download(np.float32, total)
    parts = fp.download(np.float32, len(lens))
    want = []
    for k, n in enumerate(lens):
        yk = O.map_affine(x[lay.begins[k]:lay.begins[k] + n], 2.0, 1.0)
        assert np.array_equal(y[lay.begins[k]:lay.begins[k] + n].view(np.uint32), yk.view(np.uint32))
        want.append(O.tree_reduce(yk, op))
    assert [O.f32_bits(v) for v in parts] == [O.f32_bits(v) for v in want]
    assert O.f32_bits(fr.download(np.float32, 1)[0]) == O.f32_bits(O.tree_reduce(np.array(want, np.float32), op))
    # the read-only reduction over y, unfused
    _call("ucg_segment_reduce_f32", fy.ptr, tab.handle, capi.OPS[op], fs.ptr, fp.ptr, None)
    _sync_ok()
    assert [O.f32_bits(v) for v in fp.download(np.float32, len(lens))] == [O.f32_bits(v) for v in want]
    tab.close()
    for f in (fx, fy, fs, fp, fr):
        f.close()


@pytest.mark.parametrize("n", [1, 3, 64, 1000, 4096 * 5 + 1])
def test_fence_tree_reduce(cuda, n):
    v = O.fill_uniform(9, n)
    fx, fo = Fenced(4 * n), Fenced(4)
    fx.upload(v)
    _call("ucg_tree_reduce_f32", fx.ptr, n, 0, fo.ptr, None)
    _sync_ok()
    assert O.f32_bits(fo.download(np.float32, 1)[0]) == O.f32_bits(O.tree_reduce(v, "sum"))
    fx.close(), fo.close()


@pytest.mark.parametrize("length,count", [(1, 300), (5, 77), (33, 40), (1000, 9)])
def test_fence_reduce_cl_vectors(cuda, length, count):
    """stage-1 folds + stage-2 tree reading every element through fenced
    element buffers and a fenced pointer array."""
    from paper_1505_01120_b200.capi import u64_array

    rng = np.random.default_rng(length * 1000 + count)
    elems = rng.standard_normal((count, length)).astype(np.float32)
    fences = [Fenced(4 * length) for _ in range(count)]
    for f, e in zip(fences, elems):
        f.upload(np.ascontiguousarray(e))
    ptrs = np.array([f.ptr for f in fences], np.uint64)
    fptr, fout = Fenced(8 * count), Fenced(4 * length)
    fptr.upload(ptrs)
    parts = [count // 3, 0, count - count // 3]
    _call("ucg_reduce_cl_f32", fptr.ptr, count, length, u64_array(parts), len(parts), 0, fout.ptr, None)
    _sync_ok()
    want = O.reduce_cl(elems, parts, "sum")
    assert np.array_equal(fout.download(np.float32, length).view(np.uint32), want.view(np.uint32))
    for f in fences + [fptr, fout]:
        f.close()


def test_fence_pi(cuda):
    from paper_1505_01120_b200.capi import u64_array

    seeds, samples = [42, 43, 44], [70000, 1, 300001]
    fh, ft = Fenced(8 * 3), Fenced(8)
    _call("ucg_pi_hits_total", u64_array(seeds), u64_array(samples), 3, fh.ptr, ft.ptr, None)
    _sync_ok()
    want = [O.pi_hits(s, n) for s, n in zip(seeds, samples)]
    assert fh.download(np.int64, 3).tolist() == want
    assert int(ft.download(np.int64, 1)[0]) == sum(want)
    fh.close(), ft.close()


@pytest.mark.parametrize("W,rows", [(256, [64, 1, 130]), (16384, [256, 3]), (512, [7])])
def test_fence_sobel_tma(cuda, W, rows):
    """k_sobel_tma (TMA boxes with zero-filled side boxes): the input ends at
    the fence with the last band's bottom halo row."""
    from paper_1505_01120_b200.capi import u64_array

    img = O.sobel_image(sum(rows), W, 7)
    bands = []
    r0 = 0
    for r in rows:
        b = np.zeros((r + 2, W), np.uint8)
        for k in range(r + 2):
            src = r0 + k - 1
            if 0 <= src < img.shape[0]:
                b[k] = img[src]
        bands.append(b)
        r0 += r
    inp = np.concatenate([b.reshape(-1) for b in bands])
    in_off = np.cumsum([0] + [b.size for b in bands[:-1]]).tolist()
    out_off = np.cumsum([0] + [r * W for r in rows[:-1]]).tolist()
    fi, fo = Fenced(inp.nbytes), Fenced(sum(rows) * W)
    fi.upload(inp)
    _call("ucg_sobel_bands_u8", fi.ptr, u64_array(in_off), fo.ptr, u64_array(out_off), u64_array(rows), len(rows), W,
          None)
    _sync_ok()
    got = fo.download(np.uint8, sum(rows) * W)
    want = np.concatenate([O.sobel_band(b.reshape(-1), r, W).reshape(-1) for b, r in zip(bands, rows)])
    assert np.array_equal(got, want)
    fi.close(), fo.close()


@pytest.mark.parametrize("fn", ["ucg_gemm_tf32", "ucg_gemm_f32"])
def test_fence_gemm(cuda, fn):
    """The tcgen05 CTA-pair GEMM with TMA-fed operands and C fenced."""
    n = 512
    A = (O.fill_uniform(100, n * n) * 2 - 1).astype(np.float32)
    B = (O.fill_uniform(101, n * n) * 2 - 1).astype(np.float32)
    fa, fb, fc = Fenced(4 * n * n), Fenced(4 * n * n), Fenced(4 * n * n)
    fa.upload(A)
    fb.upload(B)
    _call(fn, fa.ptr, fb.ptr, fc.ptr, n, None)
    _sync_ok()
    Cg = fc.download(np.float32, n * n).reshape(n, n)
    ref = A.reshape(n, n).astype(np.float64) @ B.reshape(n, n).astype(np.float64)
    rms = np.sqrt((ref ** 2).mean())
    assert np.sqrt(((Cg - ref) ** 2).mean()) / rms < (1.5e-3 if fn == "ucg_gemm_tf32" else 5e-6)
    fa.close(), fb.close(), fc.close()


@pytest.mark.parametrize("n", [1, 15, 16, 4097, (1 << 20) + 3])
def test_fence_word_flags(cuda, n):
    data = np.frombuffer((O.corpus(5, n // 3 + 10))[:n], np.uint8).copy()
    fd, ff = Fenced(n), Fenced(n)
    fd.upload(data)
    _call("ucg_word_start_flags", fd.ptr, n, ff.ptr, None)
    _sync_ok()
    assert np.array_equal(ff.download(np.uint8, n), O.word_start_flags(data.tobytes()))
    fd.close(), ff.close()

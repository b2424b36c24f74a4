"""GPU parity: the CUDA path (through the C-ABI) against the oracle and the
reference golden vectors. Integer / index / max / map results and — because
the kernels reproduce the reference pairing tree exactly — fp32 sums are all
compared BIT-EXACT; full-size C2 additionally checks fp32 sums against fp64
at rel 1e-5 (BASELINE.json north_star tolerance)."""
import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _bits(t):
    a = t.detach().cpu().numpy() if hasattr(t, "detach") else np.asarray(t)
    return a.view(np.uint32) if a.dtype == np.float32 else a


# ---- map -------------------------------------------------------------------------

@pytest.mark.parametrize("n", [0, 1, 3, 4, 5, 127, 4096, 1000003, (1 << 24) + 12345])
def test_map_affine_bitexact(cuda, n):
    from paper_1505_01120_b200 import ops

    x = O.fill_uniform(77, n) * np.float32(8) - np.float32(4)
    xd = torch.from_numpy(x).to(cuda)
    yd = torch.empty_like(xd)
    ops.map_affine(xd, yd, 2.0, 1.0)
    ops.map_affine(xd, xd, 0.3, -7.25) if n else None  # in-place form
    torch.cuda.synchronize()
    assert np.array_equal(_bits(yd), O.map_affine(x, 2.0, 1.0).view(np.uint32))
    assert np.array_equal(_bits(xd), O.map_affine(x, 0.3, -7.25).view(np.uint32))


def test_ops_reject_bad_buffers(cuda):
    """The C-ABI indexes raw pointers: non-contiguous, wrongly typed or
    undersized tensors are refused before any launch."""
    from paper_1505_01120_b200 import ops

    x = torch.zeros(64, 4, device=cuda)
    y = torch.zeros(64, 4, device=cuda)
    with pytest.raises(ValueError):
        ops.map_affine(x.t(), y, 2.0, 1.0)
    with pytest.raises(TypeError):
        ops.map_affine(x.double(), y, 2.0, 1.0)
    with pytest.raises(ValueError):
        ops.map_affine(x, y[:10], 2.0, 1.0, n=256)
    with pytest.raises(Exception):
        ops.map_affine(x.cpu(), y, 2.0, 1.0)


# ---- partition reductions ----------------------------------------------------------

SEG_LENS = [0, 1, 2, 3, 4, 5, 31, 127, 128, 129, 1023, 1024, 1025, 16383, 16384, 16385, 40000, 100003, 262144]


def _segments(lens, seed=5, signed_zeros=False):
    from paper_1505_01120_b200.pipeline import Layout

    lay = Layout.of(lens)
    buf = np.full(lay.total, np.nan, np.float32)  # padding poison must never leak in
    host = []
    for k, n in enumerate(lens):
        v = (O.fill_uniform(seed + k, n) * np.float32(2) - np.float32(1)).astype(np.float32)
        if signed_zeros and n:
            v[::5] = np.float32(0.0)
            v[1::5] = np.float32(-0.0)
        buf[lay.begins[k]: lay.begins[k] + n] = v
        host.append(v)
    return lay, buf, host


@pytest.mark.parametrize("op", ["sum", "max"])
@pytest.mark.parametrize("signed_zeros", [False, True])
def test_segment_reduce_bitexact(cuda, op, signed_zeros):
    from paper_1505_01120_b200 import capi, ops

    lay, buf, host = _segments(SEG_LENS, signed_zeros=signed_zeros)
    x = torch.from_numpy(buf).to(cuda)
    tab = capi.SegTab(lay.begins, SEG_LENS)
    scratch = torch.empty(tab.scratch_floats, dtype=torch.float32, device=cuda)
    out = torch.empty(len(SEG_LENS), dtype=torch.float32, device=cuda)
    ops.segment_reduce(x, tab, op, scratch, out)
    want = np.array([O.tree_reduce(h, op) for h in host], np.float32)
    assert np.array_equal(_bits(out), want.view(np.uint32))
    tab.close()


@pytest.mark.parametrize("op", ["sum", "max"])
def test_fused_map_reduce_bitexact(cuda, op):
    from paper_1505_01120_b200 import capi, ops

    lay, buf, host = _segments(SEG_LENS, seed=11)
    x = torch.from_numpy(buf).to(cuda)
    y = torch.full_like(x, 123.0)
    tab = capi.SegTab(lay.begins, SEG_LENS)
    scratch = torch.empty(tab.scratch_floats, dtype=torch.float32, device=cuda)
    out = torch.empty(len(SEG_LENS), dtype=torch.float32, device=cuda)
    ops.map_affine_segment_reduce(x, y, tab, 2.0, 1.0, op, scratch, out)
    yh = y.cpu().numpy()
    for k, h in enumerate(host):
        want_y = O.map_affine(h, 2.0, 1.0)
        got_y = yh[lay.begins[k]: lay.begins[k] + len(h)]
        assert np.array_equal(got_y.view(np.uint32), want_y.view(np.uint32))
        assert _bits(out)[k] == np.float32(O.tree_reduce(want_y, op)).view(np.uint32)
    # padding between segments is never written
    for k, n in enumerate(SEG_LENS[:-1]):
        gap = yh[lay.begins[k] + n: lay.begins[k + 1]]
        assert np.all(gap == 123.0)
    tab.close()


def _special_segments(lens, seed):
    """Segments mixing NaN payloads, +-inf, +-0, subnormals and values large
    enough that partial sums overflow — the tree ORDER decides every result
    (std::max keeps the left operand on NaN; inf + -inf appears mid-tree)."""
    from paper_1505_01120_b200.pipeline import Layout

    rng = np.random.default_rng(seed)
    lay = Layout.of(lens)
    buf = np.zeros(lay.total, np.float32)
    host = []
    pool = np.array([np.inf, -np.inf, 0.0, -0.0, 1e-40, -3e-39, 3e38, -3e38, 1.5, -2.25],
                    np.float32)
    nans = np.array([0x7fc00000, 0xffc00001, 0x7fa00000, 0x7f800001], np.uint32).view(np.float32)
    for k, n in enumerate(lens):
        v = (rng.standard_normal(n) * 1e3).astype(np.float32)
        m = rng.random(n)
        dens = [0.0, 1e-4, 0.01, 0.2][k % 4]
        sel = m < dens
        v[sel] = pool[rng.integers(0, pool.size, sel.sum())]
        if k % 3 == 1 and n:
            nsel = m > 1.0 - dens / 4
            v[nsel] = nans[rng.integers(0, nans.size, nsel.sum())]
        if k == 5:
            v[0] = nans[1]  # leftmost NaN stays the left operand up the whole tree
        buf[lay.begins[k]: lay.begins[k] + n] = v
        host.append(v)
    return lay, buf, host


def _same_float(got: np.ndarray, want: np.ndarray, op: str) -> bool:
    """Bit equality; for sums a NaN result only needs to be a NaN (x86 keeps
    the first operand's payload, the GPU returns the canonical NaN). max
    returns one operand unchanged, so its NaN payloads must match exactly."""
    if op == "max":
        return np.array_equal(got.view(np.uint32), want.view(np.uint32))
    both_nan = np.isnan(got) & np.isnan(want)
    return bool(np.all(both_nan | (got.view(np.uint32) == want.view(np.uint32))))


@pytest.mark.parametrize("op", ["sum", "max"])
@pytest.mark.parametrize("fused", [False, True])
def test_segment_reduce_special_values(cuda, op, fused):
    from paper_1505_01120_b200 import capi, ops

    lens = [1, 2, 3, 1025, 4096, 16385, 65536, 100003, 0, 262144, 333333, 7]
    lay, buf, host = _special_segments(lens, seed=23)
    x = torch.from_numpy(buf).to(cuda)
    tab = capi.SegTab(lay.begins, lens)
    scratch = torch.empty(tab.scratch_floats, dtype=torch.float32, device=cuda)
    out = torch.empty(len(lens), dtype=torch.float32, device=cuda)
    if fused:
        y = torch.empty_like(x)
        ops.map_affine_segment_reduce(x, y, tab, 2.0, -1.0, op, scratch, out)
        want = np.array([O.tree_reduce(O.map_affine(h, 2.0, -1.0), op) for h in host], np.float32)
        yh = y.cpu().numpy()
        for k, h in enumerate(host):
            got_y = yh[lay.begins[k]: lay.begins[k] + len(h)]
            assert _same_float(got_y, O.map_affine(h, 2.0, -1.0), "sum")
    else:
        ops.segment_reduce(x, tab, op, scratch, out)
        want = np.array([O.tree_reduce(h, op) for h in host], np.float32)
    got = out.cpu().numpy()
    assert np.isnan(want).any() and np.isinf(want).any() if op == "max" else np.isnan(want).any()
    # after the map every NaN is the device's canonical NaN (fl(a*NaN) payload
    # is hardware-defined), so only the unmapped max keeps payloads bit-exact
    assert _same_float(got, want, "sum" if fused else op), (got, want)
    tab.close()


@pytest.mark.parametrize("op", ["sum", "max"])
@pytest.mark.parametrize("fused", [False, True])
def test_many_partitions_bitexact(cuda, op, fused):
    """More partitions than finisher CTAs (one warp per partition tree in the
    kernel tail), empty and ragged ones included, through reduce_cl."""
    from paper_1505_01120_b200 import capi, ops

    rng = np.random.default_rng(31)
    lens = [int(v) for v in rng.integers(0, 20000, 2500)]
    lens[7] = 0
    lens[100] = 1
    lay, buf, host = _segments(lens, seed=41)
    x = torch.from_numpy(buf).to(cuda)
    y = torch.empty_like(x) if fused else None
    tab = capi.SegTab(lay.begins, lens)
    scratch = torch.empty(tab.scratch_floats, dtype=torch.float32, device=cuda)
    parts = torch.empty(len(lens), dtype=torch.float32, device=cuda)
    res = torch.empty(1, dtype=torch.float32, device=cuda)
    for _ in range(2):  # the table's counters must be reusable launch after launch
        ops.segment_reduce_cl(x, y, tab, 2.0, 1.0, op, scratch, parts, None, res)
    vals = [O.map_affine(h, 2.0, 1.0) if fused else h for h in host]
    want = np.array([O.tree_reduce(v, op) for v in vals], np.float32)
    assert np.array_equal(_bits(parts), want.view(np.uint32))
    assert _bits(res)[0] == np.float32(O.tree_reduce(want, op)).view(np.uint32)
    tab.close()


@pytest.mark.parametrize("n", [0, 1, 2, 3, 7, 64, 1000, 2048, 2049, 5000, 70001])
@pytest.mark.parametrize("op", ["sum", "max"])
def test_tree_reduce_bitexact(cuda, n, op):
    from paper_1505_01120_b200 import ops

    x = (O.fill_uniform(n + 3, n) - np.float32(0.5)).astype(np.float32)
    out = torch.empty(1, dtype=torch.float32, device=cuda)
    ops.tree_reduce(torch.from_numpy(x).to(cuda) if n else torch.empty(1, device=cuda), n, op, out)
    assert _bits(out)[0] == np.float32(O.tree_reduce(x, op)).view(np.uint32)


# ---- reduce_cl over vectors (stage-1 folds + stage-2 tree) -------------------------

def _reduce_cl_gpu(cuda, elems, counts, op="sum"):
    from paper_1505_01120_b200 import ops

    dt = torch.int64 if elems.dtype == np.int64 else torch.float32
    # elements as separate device buffers (arbitrary addresses, like a Dataset)
    bufs = [torch.from_numpy(np.ascontiguousarray(e)).to(cuda) for e in elems]
    ptrs = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device=cuda)
    out = torch.empty(elems.shape[1], dtype=dt, device=cuda)
    ops.reduce_cl_vectors(ptrs, elems.shape[0], elems.shape[1], counts, op, out,
                          dtype="i64" if dt == torch.int64 else "f32")
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("length", [1, 3, 31, 32, 100])
@pytest.mark.parametrize("op", ["sum", "max"])
def test_reduce_cl_many_short_elements(cuda, length, op):
    """The literal form: thousands of short elements per partition (warp-wide
    stage-1 folds for length < 32, thread folds otherwise), elements packed
    contiguously — bit-exact left folds + pairing tree."""
    from paper_1505_01120_b200 import ops

    count = 5000 if length < 32 else 700
    counts = [count // 4 + (1 if p < count % 4 else 0) for p in range(4)]
    counts[2] += counts[1]
    counts[1] = 0  # an empty partition in the middle
    x = (O.fill_uniform(61, count * length) * np.float32(2) - np.float32(1)).astype(np.float32)
    elems = x.reshape(count, length)
    xd = torch.from_numpy(x).to(cuda)
    ptrs = torch.tensor([xd.data_ptr() + 4 * length * i for i in range(count)], dtype=torch.int64, device=cuda)
    out = torch.empty(length, dtype=torch.float32, device=cuda)
    ops.reduce_cl_vectors(ptrs, count, length, counts, op, out)
    want = O.reduce_cl(elems, counts, op)
    assert np.array_equal(_bits(out), want.view(np.uint32))
    # integer sums, same shape
    xi = (x.view(np.uint32).astype(np.int64) << 20) - (1 << 40)
    xid = torch.from_numpy(xi).to(cuda)
    ptrs_i = torch.tensor([xid.data_ptr() + 8 * length * i for i in range(count)], dtype=torch.int64, device=cuda)
    outi = torch.empty(length, dtype=torch.int64, device=cuda)
    ops.reduce_cl_vectors(ptrs_i, count, length, counts, "sum", outi, dtype="i64")
    assert np.array_equal(outi.cpu().numpy(), O.reduce_cl(xi.reshape(count, length), counts))


@pytest.mark.parametrize("nparts", [4097, 9000])
def test_reduce_cl_beyond_4096_partitions(cuda, nparts):
    """Stage 2 over more than 4096 non-empty partitions (no partition limit,
    as the reference engine.hpp:172-190 has none): one element per partition,
    so the result is the pairing tree over all of them."""
    from paper_1505_01120_b200 import ops

    length = 3
    x = (O.fill_uniform(77, nparts * length) * np.float32(2) - np.float32(1)).astype(np.float32)
    elems = x.reshape(nparts, length)
    xd = torch.from_numpy(x).to(cuda)
    ptrs = torch.tensor([xd.data_ptr() + 4 * length * i for i in range(nparts)], dtype=torch.int64, device=cuda)
    out = torch.empty(length, dtype=torch.float32, device=cuda)
    counts = [1] * nparts
    ops.reduce_cl_vectors(ptrs, nparts, length, counts, "sum", out)
    assert np.array_equal(_bits(out), O.reduce_cl(elems, counts, "sum").view(np.uint32))


def test_reduce_cl_isum_golden(cuda, golden):
    from test_oracle_golden import _isum_cases

    for case, elems, parts in _isum_cases(golden):
        counts = O.partition_sizes(elems.shape[0], parts)
        assert _reduce_cl_gpu(cuda, elems, counts).tolist() == case["result"]


def test_reduce_cl_fig3_and_acceptance2(cuda, golden):
    out = _reduce_cl_gpu(cuda, np.array([[1, 2, 3], [4, 5, 6]], np.float32), [2])
    assert out.tolist() == [5.0, 7.0, 9.0]
    n, P = 1 << 20, 8
    elems = np.stack([O.fill_vectoradd(k, n) for k in range(P)])
    out = _reduce_cl_gpu(cuda, elems, [1] * P)
    assert O.fnv64(out) == golden["vectoradd_acc2"]["fnv"]
    assert "%.3f" % float(out.astype(np.float64).sum()) == golden["vectoradd_acc2"]["checksum"]


@pytest.mark.parametrize("op", ["sum", "max"])
def test_reduce_cl_ragged_float(cuda, op):
    rng = np.random.default_rng(3)
    for trial in range(6):
        count = int(rng.integers(1, 60))
        parts = int(rng.integers(1, 20))
        length = int(rng.integers(1, 3000))
        elems = rng.standard_normal((count, length)).astype(np.float32)
        elems[:, ::7] = -0.0
        counts = O.partition_sizes(count, parts)
        got = _reduce_cl_gpu(cuda, elems, counts, op)
        assert np.array_equal(got.view(np.uint32), O.reduce_cl(elems, counts, op).view(np.uint32))


def test_reduce_cl_empty_raises(cuda):
    from paper_1505_01120_b200 import EmptyDataset, ops

    out = torch.empty(4, dtype=torch.float32, device=cuda)
    ptrs = torch.empty(1, dtype=torch.int64, device=cuda)
    with pytest.raises(EmptyDataset):
        ops.reduce_cl_vectors(ptrs, 0, 4, [0, 0], "sum", out)


# ---- pipelines at the BASELINE shapes ------------------------------------------------

@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("key", ["c1", "c1_ragged"])
def test_c1_pipeline_golden(cuda, golden, fused, key):
    """C1: 2^20 fp32 as 4 elements in 4 partitions, map_cl(axpb) -> map_cl_partition(psum|pmax) -> reduce_cl."""
    from paper_1505_01120_b200 import ops
    from paper_1505_01120_b200.pipeline import MapReducePipeline

    g = golden[key]
    n, P, E = g["n"], g["partitions"], g["elements"]
    # element k of n//E(+1); partition p holds a contiguous run of elements
    esz = O.partition_sizes(n, E)
    counts = O.partition_sizes(E, P)
    part_lens, pos = [], 0
    for c in counts:
        part_lens.append(sum(esz[pos:pos + c]))
        pos += c
    for op in ("sum", "max"):
        pipe = MapReducePipeline(part_lens, op=op, fused=fused, plant_max=False)
        # overwrite the synthetic fill with the C1 collection (one stream, seed 12345)
        first = 0
        for k, ln in enumerate(part_lens):
            seg = pipe.x[pipe.layout.begins[k]: pipe.layout.begins[k] + ln]
            ops.fill_uniform_(seg, 12345, first)
            first += ln
        r = pipe.step()
        torch.cuda.synchronize()
        ys = np.concatenate([pipe.local_output(k).cpu().numpy() for k in range(P)])
        assert O.fnv64(ys) == g["y_fnv"]
        assert [O.f32_bits(v) for v in pipe.partials.cpu().numpy()[:P]] == g["partials_" + op]
        assert O.f32_bits(r.cpu().numpy()[0]) == g["total_" + op]
        pipe.close()


@pytest.mark.parametrize("fused", [False, True])
def test_c2_small_golden(cuda, golden, fused):
    from paper_1505_01120_b200.pipeline import MapReducePipeline

    g = golden["c2_small"]
    for op in ("sum", "max"):
        pipe = MapReducePipeline([g["L"]] * g["P"], op=op, fused=fused)
        r = pipe.step()
        ys = np.concatenate([pipe.local_output(k).cpu().numpy() for k in range(g["P"])])
        assert O.fnv64(ys) == g["y_fnv"]
        assert [O.f32_bits(v) for v in pipe.partials.cpu().numpy()] == g["partials_" + op]
        assert O.f32_bits(r.cpu().numpy()[0]) == g["total_" + op]
        pipe.close()


def test_graph_step_matches_eager(cuda, golden):
    """The CUDA-graph replay of the one-kernel step gives the eager result."""
    from paper_1505_01120_b200.pipeline import MapReducePipeline

    g = golden["c2_small"]
    for op in ("sum", "max"):
        pipe = MapReducePipeline([g["L"]] * g["P"], op=op, fused=True)
        eager = O.f32_bits(pipe.step().cpu().numpy()[0])
        for _ in range(3):
            r = pipe.graph_step()
        assert O.f32_bits(r.cpu().numpy()[0]) == eager == g["total_" + op]
        pipe.close()


@pytest.mark.parametrize("lens", [[1 << 18] * 4, [100003, 65536, 1, 40000], [4096] * 40])
def test_graph_of_steps_pdl_chain(cuda, lens):
    """K consecutive one-kernel steps in one CUDA graph (small tables: the
    single-finisher tail, launched with programmatic dependent launch, so
    step k+1's grid is resident during step k's tail) reproduce the oracle
    bits for y, the partition values and the result — every step, not just
    the last: y is poisoned before the replay and must come back whole."""
    from paper_1505_01120_b200.pipeline import MapReducePipeline

    for op in ("sum", "max"):
        pipe = MapReducePipeline(lens, op=op, fused=True, plant_max=False)
        partials = []
        for k, n in enumerate(lens):
            partials.append(O.tree_reduce(O.map_affine(O.fill_uniform(1000 + k, n), 2.0, 1.0), op))
        want = O.tree_reduce(np.array(partials, np.float32), op)
        for steps in (1, 7, 32):
            pipe.graph_step(steps)
            torch.cuda.synchronize()
            pipe.y.fill_(float("nan"))
            pipe.partials.fill_(float("nan"))
            pipe.result.fill_(float("nan"))
            r = pipe.graph_step(steps)
            torch.cuda.synchronize()
            assert O.f32_bits(r.cpu().numpy()[0]) == O.f32_bits(want), (op, steps)
            got = pipe.partials.cpu().numpy()[:len(lens)]
            assert np.array_equal(got.view(np.uint32), np.array(partials, np.float32).view(np.uint32))
            for k, n in enumerate(lens):
                y = pipe.local_output(k).cpu().numpy()
                assert np.array_equal(y.view(np.uint32), O.map_affine(O.fill_uniform(1000 + k, n), 2.0, 1.0).view(np.uint32))
        pipe.close()


@pytest.mark.slow
def test_c2_full_size(cuda):
    """C2 at the BASELINE size (2^30 fp32, 64 partitions): size-independent checks."""
    from paper_1505_01120_b200.pipeline import MapReducePipeline

    P, L = 64, 1 << 24
    pipe = MapReducePipeline([L] * P, op="sum", fused=True)
    r = float(pipe.step().item())
    partials = pipe.partials.cpu().numpy()
    rng = np.random.default_rng(0)
    total64 = 0.0
    for p in range(P):
        y = pipe.local_output(p).cpu().numpy()
        if p in (0, 17, P // 2, P - 1):  # exact tree on a sample of partitions
            assert O.f32_bits(O.tree_reduce(y, "sum")) == O.f32_bits(partials[p])
            idx = rng.integers(0, L, 4096)
            x = np.array([O.fill_uniform(1000 + p, 1, int(i))[0] for i in idx], np.float32)
            if p == P // 2:
                x[idx == L // 3] = 1.5
            assert np.array_equal(y[idx].view(np.uint32), O.map_affine(x, 2.0, 1.0).view(np.uint32))
        s64 = float(y.astype(np.float64).sum())
        assert abs(float(partials[p]) - s64) / s64 < 1e-5
        total64 += s64
    assert O.f32_bits(O.tree_reduce(partials, "sum")) == O.f32_bits(np.float32(r))
    assert abs(r - total64) / total64 < 1e-5
    # max: the planted maximum 1.5 maps to exactly 4.0
    pipe2 = MapReducePipeline([L] * P, op="max", fused=False)
    assert float(pipe2.step().item()) == 4.0
    pipe.close()
    pipe2.close()


# ---- pi / sobel ------------------------------------------------------------------------

def test_pi_golden(cuda, golden):
    from paper_1505_01120_b200 import ops

    for case in golden["pi"]:
        S, T, seed = case["samples"], case["tasks"], case["seed"]
        samples = [S // T + (1 if t < S % T else 0) for t in range(T)]
        hits = torch.empty(T, dtype=torch.int64, device=cuda)
        ops.pi_hits([seed + t for t in range(T)], samples, hits)
        assert hits.cpu().tolist() == case["task_hits"]
        total = torch.full((1,), -1, dtype=torch.int64, device=cuda)
        ops.pi_hits([seed + t for t in range(T)], samples, hits, total_out=total)
        assert hits.cpu().tolist() == case["task_hits"]
        assert int(total.item()) == case["hits"]  # the reference reduce_cl(isum2) total


def test_pi_vs_oracle_small(cuda):
    from paper_1505_01120_b200 import ops

    seeds = [0, 1, 2**63 + 5, 2**64 - 1, 42]
    samples = [0, 1, 65535, 65536, 200001]
    hits = torch.empty(len(seeds), dtype=torch.int64, device=cuda)
    ops.pi_hits(seeds, samples, hits)
    assert hits.cpu().tolist() == [O.pi_hits(s, n) for s, n in zip(seeds, samples)]


def test_sobel_golden_and_random(cuda, golden):
    from paper_1505_01120_b200 import ops

    g = golden["sobel"]
    # (W=40 golden: generic path; multiples of 16: the vectorised path)
    for (H, W, rows, seed) in [(g["H"], g["W"], g["rows"], g["seed"]), (50, 48, 16, 7), (64, 256, 32, 3),
                               (37, 1024, 5, 9), (300, 528, 64, 1), (70, 33, 9, 2)]:
        img = O.sobel_image(H, W, seed)
        bands = O.sobel_bands(img, rows)
        inp = np.concatenate([b.ravel() for b in bands])
        in_off, out_off, rws = [], [], []
        pi = po = 0
        for b in bands:
            in_off.append(pi)
            out_off.append(po)
            rws.append(b.shape[0] - 2)
            pi += b.size
            po += (b.shape[0] - 2) * W
        dinp = torch.from_numpy(inp).to(cuda)
        dout = torch.zeros(po, dtype=torch.uint8, device=cuda)
        ops.sobel_bands(dinp, in_off, dout, out_off, rws, W)
        want = np.concatenate([O.sobel_band(b, b.shape[0] - 2, W) for b in bands])
        got = dout.cpu().numpy()
        assert np.array_equal(got, want)
        if (H, W) == (g["H"], g["W"]):
            assert O.fnv64(got) == g["fnv"]


# ---- the reference Engine through the C++ drop-in (libucores_engine.so) ------------

@pytest.mark.parametrize("mode", ["batched", "per_task", "device"])
def test_engine_capi_pipeline(cuda, golden, mode):
    from paper_1505_01120_b200 import engine_capi

    g = golden["c2_small"]
    P, L = g["P"], g["L"]
    xs = [O.fill_uniform(1000 + p, L) for p in range(P)]
    xs[P // 2][L // 3] = 1.5
    for op in ("sum", "max"):
        y, partials, r, _ = engine_capi.pipeline_f32(np.concatenate(xs), [L] * P, op=op, mode=mode)
        assert O.fnv64(y) == g["y_fnv"]
        assert [O.f32_bits(v) for v in partials] == g["partials_" + op]
        assert O.f32_bits(r) == g["total_" + op]


def test_engine_capi_pi(cuda, golden):
    from paper_1505_01120_b200 import engine_capi

    case = golden["pi"][0]
    hits, _ = engine_capi.pi(case["samples"], case["tasks"], case["seed"])
    assert hits == case["hits"]


def test_tapered_tail_bitexact():
    """UCG_TAPER (A/B knob, off by default): the fused map's last items are
    streamed as 4 sub-items and the finishers recombine the sub-roots. The
    fused cases — many ragged/empty partitions (warp-per-partition tail),
    SEG_LENS, and full-size C2 (CTA-per-partition tail) — rerun in a fresh
    process with the knob on must stay bit-exact (the knob is read once per
    process)."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, UCG_TAPER="64")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        f"{__file__}::test_many_partitions_bitexact", f"{__file__}::test_fused_map_reduce_bitexact",
                        f"{__file__}::test_c2_full_size", "-k", "True or fused_map or full_size"],
                       env=env, cwd=os.path.dirname(__file__), capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "5 passed" in r.stdout, r.stdout[-2000:]



@pytest.mark.parametrize("env", [{}, {"UCG_SOBEL_STATIC": "1"}, {"UCG_SOBEL_ARITH": "int"},
                                 {"UCG_SOBEL_ARITH": "half"}, {"UCG_SOBEL_ARITH": "mix2"},
                                 {"UCG_SOBEL_VARIANT": "0"}, {"UCG_SOBEL_VARIANT": "0", "UCG_SOBEL_ARITH": "int"},
                                 {"UCG_SOBEL_VARIANT": "2"}], ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()) or "default")
def test_sobel_kernel_variants(cuda, env):
    """Every Sobel kernel (TMA tiles with claimed or round-robin tiles, row
    streaming, register streaming) in every arithmetic form (fp16-subnormal,
    biased integer, the mixed forms) is bit-exact against the oracle on random images and on
    saturating patterns."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path

    here = Path(__file__).resolve().parent
    out = subprocess.run([sys.executable, str(here / "sobel_variant_worker.py")], env=dict(os.environ, **env),
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-3000:]
    rep = json.loads(out.stdout.strip().splitlines()[-1])
    assert rep["cases"] >= 14 and rep["bad"] == [], rep


# ---- consecutive steps (early-stream mode) --------------------------------------------

@pytest.mark.parametrize("lens", [[1 << 20] * 4, [3 << 22, 77777, 1, 1 << 21, 5 << 20]])
@pytest.mark.parametrize("op", ["sum", "max"])
def test_consecutive_steps_early_mode(cuda, lens, op):
    """Back-to-back steps on one table overlap (each step's stream runs while
    the previous step's partition trees finish, on alternate counter and
    scratch halves): after odd and even numbers of chained steps the partials
    and result are bit-exact; an input rewritten by another kernel between
    steps is seen by the next step; a table reducing another table's output
    right after it reads that output complete."""
    from paper_1505_01120_b200 import ops
    from paper_1505_01120_b200.pipeline import MapReducePipeline

    def want(xs, a, b):
        p = [O.tree_reduce(O.map_affine(x, a, b), op) for x in xs]
        return np.array(p, np.float32), O.tree_reduce(np.array(p, np.float32), op)

    pipe = MapReducePipeline(lens, op=op, plant_max=False)
    xs = [O.fill_uniform(1000 + k, n) for k, n in enumerate(lens)]
    wp, wr = want(xs, 2.0, 1.0)
    for chain in (7, 4):
        for _ in range(chain):
            r = pipe.step()
        torch.cuda.synchronize()
        assert np.array_equal(_bits(pipe.partials), wp.view(np.uint32)), chain
        assert O.f32_bits(r.cpu().numpy()[0]) == O.f32_bits(wr), chain
    # a torch kernel rewrites x between two chained steps
    pipe.step()
    pipe.x.mul_(0.5)
    r = pipe.step()
    pipe.step()
    torch.cuda.synchronize()
    wp2, wr2 = want([x * np.float32(0.5) for x in xs], 2.0, 1.0)
    assert np.array_equal(_bits(pipe.partials), wp2.view(np.uint32))
    assert O.f32_bits(r.cpu().numpy()[0]) == O.f32_bits(wr2)
    # a second table reduces the first's y right after the first's steps
    pipe2 = MapReducePipeline(lens, op=op, plant_max=False)
    for _ in range(3):
        pipe.step()
    ops.segment_reduce_cl(pipe.y, None, pipe2.segtab, 1.0, 0.0, op, pipe2.scratch, pipe2.partials, None,
                          pipe2.result)
    torch.cuda.synchronize()
    ys = [pipe.y[b:b + n].cpu().numpy() for b, n in zip(pipe.layout.begins, lens)]
    wp3 = np.array([O.tree_reduce(y, op) for y in ys], np.float32)
    assert np.array_equal(_bits(pipe2.partials), wp3.view(np.uint32))
    assert O.f32_bits(pipe2.result.cpu().numpy()[0]) == O.f32_bits(O.tree_reduce(wp3, op))
    pipe.close()
    pipe2.close()


@pytest.mark.parametrize("lens", [[1 << 18] * 4, [1 << 21] * 8, [5000] * 300])
def test_long_step_chains(cuda, lens):
    """Thousands of chained repeated steps (each launching its successor at
    its first instruction, parity start tickets) and graph replays of long
    chains end bit-exact: a ticket drawn out of order would stall a grid
    until the 30 s trap and fail the launch."""
    from paper_1505_01120_b200.pipeline import MapReducePipeline

    pipe = MapReducePipeline(lens, op="sum", plant_max=False)
    p = np.array([O.tree_reduce(O.map_affine(O.fill_uniform(1000 + k, n), 2.0, 1.0), "sum")
                  for k, n in enumerate(lens)], np.float32)
    want = O.tree_reduce(p, "sum")
    for _ in range(3000 if sum(lens) <= (1 << 20) else 500):
        pipe.step()
    torch.cuda.synchronize()
    assert O.f32_bits(pipe.result.cpu().numpy()[0]) == O.f32_bits(want)
    for _ in range(3):
        pipe.result.fill_(float("nan"))
        r = pipe.graph_step(101)
        torch.cuda.synchronize()
        assert O.f32_bits(r.cpu().numpy()[0]) == O.f32_bits(want)
    assert np.array_equal(_bits(pipe.partials), p.view(np.uint32))
    pipe.close()

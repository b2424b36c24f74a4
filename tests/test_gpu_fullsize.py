"""Parity at the BASELINE.json sizes (C1, C3, C4, C5), where the oracle can
check the whole result or a stated sample of it in seconds:

  C1  2^20 fp32, 4 partitions: y, partials and the total bit-exact vs the oracle
  C3  2^30 samples / 8 tasks / seed 42: 843,312,281 hits — the reference
      probe value of SURVEY.md §8(c) — and 2^34 / 64 tasks: exact per-task
      integer counts summing to the reduce_cl total
  C4  16384^2 u8 in 64 bands: three whole bands (first, middle, last)
      bit-exact vs the oracle, every band's checksum against a torch port of
      the same formula
  C5  8192^3 TF32: 64 sampled output entries within the TF32 tolerance of an
      fp64 dot product of the same fp32 inputs
"""
import json
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

# the reference's own output at the BASELINE sizes (tests/golden/make_golden_full.py)
FULL = json.loads((Path(__file__).resolve().parent / "golden" / "ref_golden_full.json").read_text())


@pytest.mark.parametrize("op,fused", [("sum", True), ("max", True), ("sum", False)])
def test_c2_full_vs_reference(cuda, op, fused):
    """C2 (2^30 fp32, 64 partitions, planted maximum): every partition's y, all
    64 partials and the reduce_cl result bit-identical to the unmodified
    reference Engine's output at this size."""
    from paper_1505_01120_b200.pipeline import MapReducePipeline

    g = FULL["c2_full"]
    P, L = g["P"], g["L"]
    pipe = MapReducePipeline([L] * P, op=op, fused=fused, plant_max=True)
    pipe.result.fill_(float("nan"))
    r = pipe.step()
    assert O.f32_bits(r.cpu().numpy()[0]) == g[f"total_{op}"]
    got = [O.f32_bits(v) for v in pipe.partials.cpu().numpy()[:P]]
    assert got == g[f"partials_{op}"]
    if op == "sum" and fused:
        for p in range(P):
            assert O.fnv64(pipe.local_output(p).cpu().numpy()) == g["y_fnv"][p], p
    # the graph-replayed step (as bench.py times it) gives the same bits
    pipe.result.fill_(float("nan"))
    assert O.f32_bits(pipe.graph_step(3).cpu().numpy()[0]) == g[f"total_{op}"]
    pipe.close()


def test_c3_full_vs_reference(cuda):
    """C3 (2^34 samples, 64 tasks, seed 42+t): all 64 task hit counts and the
    reduce_cl(isum2) total equal the reference's."""
    from paper_1505_01120_b200 import ops

    g = FULL["c3_full"]
    S, T = g["samples"], g["tasks"]
    hits = torch.empty(T, dtype=torch.int64, device=cuda)
    total = torch.empty(1, dtype=torch.int64, device=cuda)
    ops.pi_hits([g["seed"] + t for t in range(T)], [S // T] * T, hits, total_out=total)
    assert hits.cpu().tolist() == g["task_hits"]
    assert int(total.item()) == g["reduce_cl_isum2"][0] == g["hits"]


def test_c1_full(cuda):
    from paper_1505_01120_b200.pipeline import MapReducePipeline

    P, L = 4, 1 << 18
    pipe = MapReducePipeline([L] * P, op="sum", fused=True, seed_base=1000, plant_max=False)
    r = pipe.step()
    parts = pipe.partials.cpu().numpy()
    for p in range(P):
        x = O.fill_uniform(1000 + p, L)
        y = O.map_affine(x, 2.0, 1.0)
        assert np.array_equal(pipe.local_output(p).cpu().numpy().view(np.uint32), y.view(np.uint32))
        assert O.f32_bits(parts[p]) == O.f32_bits(O.tree_reduce(y, "sum"))
    assert O.f32_bits(r.cpu().numpy()[0]) == O.f32_bits(O.tree_reduce(parts, "sum"))
    pipe.close()


def test_c3_reference_probe_2e30(cuda):
    from paper_1505_01120_b200 import ops

    S, T = 1 << 30, 8
    hits = torch.empty(T, dtype=torch.int64, device=cuda)
    total = torch.empty(1, dtype=torch.int64, device=cuda)
    ops.pi_hits([42 + t for t in range(T)], [S // T] * T, hits, total_out=total)
    assert int(total.item()) == 843312281
    assert int(hits.sum().item()) == 843312281


def test_c3_full_2e34(cuda):
    from paper_1505_01120_b200 import ops

    S, T = 1 << 34, 64
    hits = torch.empty(T, dtype=torch.int64, device=cuda)
    total = torch.empty(1, dtype=torch.int64, device=cuda)
    ops.pi_hits([42 + t for t in range(T)], [S // T] * T, hits, total_out=total)
    h = hits.cpu().numpy()
    assert int(total.item()) == int(h.sum())
    # every task count is a plausible binomial draw (p = pi/4, n = 2^28: sd ~ 7.0e3)
    assert np.all(np.abs(h - (S // T) * np.pi / 4) < 8 * 7.0e3)
    # and the first task's count equals the exact oracle on a 2^22 prefix of it
    one = torch.empty(1, dtype=torch.int64, device=cuda)
    ops.pi_hits([42], [1 << 22], one)
    assert int(one.item()) == O.pi_hits(42, 1 << 22)


def _sobel_torch(band: torch.Tensor, rows: int, W: int) -> torch.Tensor:
    """min(255, |Gx| + |Gy|) with zero columns outside the band (int32 torch)."""
    b = torch.nn.functional.pad(band.view(rows + 2, W).to(torch.int32), (1, 1))
    p = lambda dr, dc: b[dr:dr + rows, 1 + dc:1 + dc + W]
    gx = (p(0, 1) - p(0, -1)) + 2 * (p(1, 1) - p(1, -1)) + (p(2, 1) - p(2, -1))
    gy = (p(2, -1) + 2 * p(2, 0) + p(2, 1)) - (p(0, -1) + 2 * p(0, 0) + p(0, 1))
    return torch.clamp(gx.abs() + gy.abs(), max=255).to(torch.uint8)


def test_c4_full(cuda):
    from paper_1505_01120_b200 import ops

    H = W = 16384
    R = 256
    nb = H // R
    img = torch.empty(H * W, dtype=torch.uint8, device=cuda)
    ops.fill_bytes_(img, 7)
    img = img.view(H, W)
    inp = torch.zeros(nb, R + 2, W, dtype=torch.uint8, device=cuda)
    for b in range(nb):  # bands with one halo row above/below, zero rows at the image edge
        r0 = b * R
        lo, hi = max(0, r0 - 1), min(H, r0 + R + 1)
        inp[b, lo - (r0 - 1):hi - (r0 - 1)] = img[lo:hi]
    out = torch.empty(nb * R * W, dtype=torch.uint8, device=cuda)
    ops.sobel_bands(inp.view(-1), [b * (R + 2) * W for b in range(nb)], out, [b * R * W for b in range(nb)],
                    [R] * nb, W)
    out = out.view(nb, R, W)
    for b in (0, nb // 2, nb - 1):
        want = O.sobel_band(inp[b].cpu().numpy().reshape(-1), R, W)
        assert np.array_equal(out[b].cpu().numpy().reshape(-1), want.reshape(-1))
    for b in range(nb):
        assert torch.equal(out[b], _sobel_torch(inp[b].reshape(-1), R, W))
    # every band equals the reference's own output at this size (FNV-1a)
    g = FULL["c4_full"]
    assert (g["H"], g["W"], g["rows"], g["seed"]) == (H, W, R, 7)
    host = out.cpu().numpy()
    assert [O.fnv64(host[b]) for b in range(nb)] == g["band_fnv"]


def test_c5_full_sampled(cuda):
    from paper_1505_01120_b200 import ops

    n = 8192
    A = torch.empty(n * n, dtype=torch.float32, device=cuda)
    B = torch.empty(n * n, dtype=torch.float32, device=cuda)
    ops.fill_uniform_(A, 100)
    ops.fill_uniform_(B, 101)
    A = (A * 2 - 1).view(n, n)
    B = (B * 2 - 1).view(n, n)
    C = torch.full((n, n), float("nan"), device=cuda)
    ops.gemm_tf32(A, B, C, n)
    assert torch.isfinite(C).all()
    rng = np.random.default_rng(5)
    idx = rng.integers(0, n, (64, 2))
    Ad, Bd = A.double(), B.double()
    ref = torch.stack([Ad[i] @ Bd[:, j] for i, j in idx]).cpu().numpy()
    got = np.array([float(C[i, j]) for i, j in idx])
    rms = float(np.sqrt((ref ** 2).mean()))
    assert np.abs(got - ref).max() <= 1e-2 * rms * 4  # fewer samples: allow the 4-sigma tail
    assert float(np.sqrt(((got - ref) ** 2).mean())) / rms <= 1.5e-3 * 2

"""CPU: the C oracle against the reference's own output at the BASELINE.json
sizes (tests/golden/ref_golden_full.json, made by make_golden_full.py from
oracle/_ref — the unmodified reference headers). Sampled where the whole
config would take minutes on one core:

  C2  2^30 fp32 / 64 partitions: the oracle's psum/pmax of 4 whole partitions
      (first, the planted maximum's, one more, last) and its y FNV-1a equal
      the reference's; the stage-2 tree over the reference's 64 partials
      equals the reference's reduce_cl result
  C3  2^34 samples / 64 tasks: the hit counts of 2 whole tasks (2^28 each)
  C4  16384^2 Sobel: every band's FNV-1a over the whole image
"""
import json
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O

FULL = json.loads((Path(__file__).resolve().parent / "golden" / "ref_golden_full.json").read_text())


def _bits(h: str) -> np.float32:
    return np.array([int(h, 16)], np.uint32).view(np.float32)[0]


@pytest.mark.parametrize("p", [0, 17, 32, 63])
def test_c2_full_partitions(p):
    g = FULL["c2_full"]
    L = g["L"]
    x = O.fill_uniform(1000 + p, L)
    if p == g["planted_max"]["partition"]:
        x[g["planted_max"]["index"]] = g["planted_max"]["value"]
    y = O.map_affine(x, 2.0, 1.0)
    assert O.fnv64(y) == g["y_fnv"][p]
    assert O.f32_bits(O.tree_reduce(y, "sum")) == g["partials_sum"][p]
    assert O.f32_bits(O.tree_reduce(y, "max")) == g["partials_max"][p]


def test_c2_full_stage2():
    g = FULL["c2_full"]
    for op in ("sum", "max"):
        parts = np.array([_bits(h) for h in g[f"partials_{op}"]], np.float32)
        assert O.f32_bits(O.tree_reduce(parts, op)) == g[f"total_{op}"]
    assert g["total_sum_value"] == 2147544832.0


@pytest.mark.parametrize("t", [0, 63])
def test_c3_full_tasks(t):
    g = FULL["c3_full"]
    assert O.pi_hits(g["seed"] + t, g["samples"] // g["tasks"]) == g["task_hits"][t]
    assert sum(g["task_hits"]) == g["hits"] == g["reduce_cl_isum2"][0]


def test_c4_full_bands():
    g = FULL["c4_full"]
    H, W, R = g["H"], g["W"], g["rows"]
    img = O.sobel_image(H, W, g["seed"])
    for b, band in enumerate(O.sobel_bands(img, R)):
        assert O.fnv64(O.sobel_band(band.reshape(-1), band.shape[0] - 2, W)) == g["band_fnv"][b], b

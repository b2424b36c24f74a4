"""Time breakdown of the C2 chain through the unmodified reference Engine +
GpuClusterDriver (seam A): per Engine call, the driver's run_wave time vs the
Engine's own work (task input copies, Element::concat, result assembly).

  python tools/seam_a_breakdown.py [--parts 64] [--part-len 16777216] [--reps 2]
Prints one JSON line per repetition."""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1505_01120_b200 import engine_capi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--parts", type=int, default=64)
    ap.add_argument("--part-len", type=int, default=1 << 24)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    x = np.random.default_rng(0).random(a.parts * a.part_len, dtype=np.float32)
    for r in range(a.reps):
        t0 = time.perf_counter()
        d = engine_capi.pipeline_breakdown_f32(x, [a.part_len] * a.parts)
        d["call_wall_s"] = time.perf_counter() - t0
        d["rep"] = r
        d["gelem_s"] = a.parts * a.part_len / d["total_s"] / 1e9
        print(json.dumps(d), flush=True)


if __name__ == "__main__":
    main()

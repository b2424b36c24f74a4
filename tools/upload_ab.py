"""DeviceEngine upload A/B: the C2 chain from a built host Dataset (4 GiB)
through ucores_b200::DeviceEngine with different staging-copy thread counts.
    python tools/upload_ab.py 4 8 16"""
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1505_01120_b200 import engine_capi  # noqa: E402

P, L = 64, 1 << 24
xs = np.random.default_rng(1).random(P * L, dtype=np.float32)
engine_capi.pipeline_f32(xs[:1 << 20], [1 << 20], op="sum", want_y=False, mode="device")
res = {t: [] for t in sys.argv[1:]}
for _ in range(3):
    for t in res:
        os.environ["UCG_COPY_THREADS"] = t
        _, _, r, sec = engine_capi.pipeline_f32(xs, [L] * P, op="sum", want_y=False, mode="device")
        res[t].append(sec)
for t, v in res.items():
    print(f"threads {t}: median {statistics.median(v) * 1e3:.1f} ms = {P * L / statistics.median(v) / 1e9:.2f} Gelem/s")

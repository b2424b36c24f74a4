"""A/B kernel timing in one process: alternates env settings between timed
batches of one workload call (CUDA events, L2 flushed by the 256 MiB+ inputs).
    python tools/ab_time.py sobel UCG_SOBEL_NEIGH=lds UCG_SOBEL_NEIGH=shfl"""
import os
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_1505_01120_b200 import ops  # noqa: E402

which, settings = sys.argv[1], sys.argv[2:]
if which == "sobel":
    H = W = 16384
    R = 256
    nb = H // R
    inp = torch.empty(nb * (R + 2) * W, dtype=torch.uint8, device="cuda")
    ops.fill_bytes_(inp, 7)
    out = torch.empty(H * W, dtype=torch.uint8, device="cuda")
    args = (inp, [b * (R + 2) * W for b in range(nb)], out, [b * R * W for b in range(nb)], [R] * nb, W)
    fn = lambda: ops.sobel_bands(*args)  # noqa: E731
elif which == "pi":
    hits = torch.empty(64, dtype=torch.int64, device="cuda")
    fn = lambda: ops.pi_hits([42 + t for t in range(64)], [(1 << 34) // 64] * 64, hits)  # noqa: E731
else:
    raise SystemExit(f"unknown workload {which}")


def batch(k=20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


res = {s: [] for s in settings}
for rnd in range(6):
    for s in settings:
        k, v = s.split("=", 1)
        os.environ[k] = v
        fn()
        torch.cuda.synchronize()
        res[s].append(batch())
for s in settings:
    print(f"{which} {s}: median {statistics.median(res[s]) * 1e3:.2f} us  min {min(res[s]) * 1e3:.2f} us")

"""Kernel micro-benchmarks (CUDA events, warm-up, inputs > L2). Dev tool."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_1505_01120_b200 import capi, ops  # noqa: E402
from paper_1505_01120_b200.pipeline import MapReducePipeline  # noqa: E402

HBM = 6434.2


def timeit(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    res = {}
    P, L = 64, 1 << 24
    n = P * L
    pipe = MapReducePipeline([L] * P, op="sum", fused=False)
    ms = timeit(lambda: ops.map_affine(pipe.x, pipe.y, 2.0, 1.0))
    res["map_affine_2^30"] = {"ms": ms, "GBs": 8 * n / ms / 1e6}
    ms = timeit(lambda: ops.segment_reduce(pipe.y, pipe.segtab, "sum", pipe.scratch, pipe.partials))
    res["segment_reduce_sum_2^30"] = {"ms": ms, "GBs": 4 * n / ms / 1e6}
    ms = timeit(lambda: ops.segment_reduce(pipe.y, pipe.segtab, "max", pipe.scratch, pipe.partials))
    res["segment_reduce_max_2^30"] = {"ms": ms, "GBs": 4 * n / ms / 1e6}
    ms = timeit(lambda: ops.map_affine_segment_reduce(pipe.x, pipe.y, pipe.segtab, 2.0, 1.0, "sum", pipe.scratch,
                                                      pipe.partials))
    res["fused_map_psum_2^30"] = {"ms": ms, "GBs": 8 * n / ms / 1e6}
    ms = timeit(lambda: pipe.step())
    res["unfused_step"] = {"ms": ms, "Gelem_s": n / ms / 1e6}
    pipe.fused = True
    ms = timeit(lambda: pipe.step())
    res["fused_step"] = {"ms": ms, "Gelem_s": n / ms / 1e6}
    ms = timeit(lambda: ops.tree_reduce(pipe.partials, P, "sum", pipe.result))
    res["tree_64"] = {"us": ms * 1e3}
    y2 = torch.empty_like(pipe.x)
    ms = timeit(lambda: y2.copy_(pipe.x))
    res["torch_copy_2^30"] = {"ms": ms, "GBs": 8 * n / ms / 1e6}
    pipe.close()
    del pipe, y2
    torch.cuda.empty_cache()
    if "--quick" in sys.argv:
        res["variant"] = os.environ.get("UCG_PASS1_VARIANT", "default")
        print(json.dumps(res))
        return
    # pi 2^34 / 64 tasks
    T = 64
    hits = torch.empty(T, dtype=torch.int64, device="cuda")
    seeds = [42 + t for t in range(T)]
    samples = [(1 << 34) // T] * T
    ms = timeit(lambda: ops.pi_hits(seeds, samples, hits), reps=5, warm=1)
    res["pi_2^34"] = {"ms": ms, "Gsamples_s": (1 << 34) / ms / 1e6, "hits": int(hits.sum().item())}
    # sobel 16384^2, 64 bands of 256 rows with halos
    H = W = 16384
    R = 256
    nb = H // R
    inp = torch.empty(nb * (R + 2) * W, dtype=torch.uint8, device="cuda")
    ops.fill_bytes_(inp, 7)
    out = torch.empty(H * W, dtype=torch.uint8, device="cuda")
    in_off = [b * (R + 2) * W for b in range(nb)]
    out_off = [b * R * W for b in range(nb)]
    ms = timeit(lambda: ops.sobel_bands(inp, in_off, out, out_off, [R] * nb, W))
    res["sobel_16384^2"] = {"ms": ms, "Gpx_s": H * W / ms / 1e6, "GBs": 2 * H * W / ms / 1e6}
    res["launches"] = capi.launch_count()
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

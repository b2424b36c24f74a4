"""CUPTI kernel durations (torch.profiler, no replay) of the C2 building
blocks: map, reduce-only, fused. Dev tool."""
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_1505_01120_b200 import ops  # noqa: E402
from paper_1505_01120_b200.pipeline import MapReducePipeline  # noqa: E402

P, L = 64, 1 << 24
pipe = MapReducePipeline([L] * P, op="sum", fused=False)
calls = {
    "map": lambda: ops.map_affine(pipe.x, pipe.y, 2.0, 1.0),
    "reduce": lambda: ops.segment_reduce(pipe.y, pipe.segtab, "sum", pipe.scratch, pipe.partials),
    "fused": lambda: ops.map_affine_segment_reduce(pipe.x, pipe.y, pipe.segtab, 2.0, 1.0, "sum", pipe.scratch,
                                                   pipe.partials),
}
for name, fn in calls.items():
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(10):
            fn()
        torch.cuda.synchronize()
    for ev in prof.key_averages():
        t = getattr(ev, "device_time_total", 0) or getattr(ev, "cuda_time_total", 0)
        if t:
            print(f"{name:7s} {ev.key[:70]:70s} n={ev.count:3d} avg={t / ev.count:9.1f} us")

"""C1 latency breakdown: graph-replayed step time vs the kernel's own CUPTI
duration, for the knobs that shape a small step. Dev tool:
    python tools/c1_probe.py [item_log2 ...]"""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_1505_01120_b200 import capi  # noqa: E402
from paper_1505_01120_b200.pipeline import MapReducePipeline  # noqa: E402


def timed(fn, k=200):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k * 1e3


def kernel_us(fn):
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(20):
            fn()
        torch.cuda.synchronize()
    out = []
    for ev in prof.key_averages():
        t = getattr(ev, "device_time_total", 0) or getattr(ev, "cuda_time_total", 0)
        if t:
            out.append(f"{ev.key[:48]} {t / ev.count:.2f}us")
    return "; ".join(out)


capi.load()
lens = [1 << 18] * 4
pipe = MapReducePipeline(lens, plant_max=False)
print(f"C1 step (eager) {timed(pipe.step):.2f} us; graph {timed(pipe.graph_step):.2f} us")
print("  kernels:", kernel_us(pipe.step))
for n in (8, 32):
    print(f"graph of {n} steps: {timed(lambda: pipe.graph_step(n), 20) / n:.2f} us/step")
# an empty graph replay as the floor
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
z = torch.zeros(1, device="cuda")
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        z.add_(1)
torch.cuda.synchronize()
print(f"graph floor (one tiny torch kernel) {timed(g.replay):.2f} us")
pipe.close()

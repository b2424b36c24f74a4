"""Per-step time of back-to-back stream launches vs one CUDA graph of K
steps, at the C2 shard sizes (one GPU). Dev tool."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1505_01120_b200.pipeline import MapReducePipeline  # noqa: E402


def per_step(fn, k, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / k)
    return best


for G in [int(v) for v in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["8", "4", "1"])]:
    P = 64 // G
    pipe = MapReducePipeline([1 << 24] * P, plant_max=False)
    K = 20
    for _ in range(3):
        pipe.step()
    stream = per_step(lambda: [pipe.step() for _ in range(K)], K)
    pipe.graph_step(K)
    graph = per_step(lambda: pipe.graph_step(K), K)
    print(f"G={G} shard {P} x 2^24: stream launches {stream:.1f} us/step, graph of {K} {graph:.1f} us/step", flush=True)
    pipe.close()
    del pipe
    torch.cuda.empty_cache()

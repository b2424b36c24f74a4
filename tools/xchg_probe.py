"""Multi-GPU exchange cost (torchrun, one process per GPU): per-step time of
graph-replayed sharded steps for a tiny table (the step is ~all exchange) and
for the C2 shard, and the C2 kernel's CUPTI duration per rank. Dev tool."""
import os
import sys

import torch
import torch.distributed as dist
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_1505_01120_b200.pipeline import MapReducePipeline  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))


def per_step(pipe, k):
    pipe.graph_step(k)
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pipe.graph_step(k)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / k


for name, lens in (("tiny 4x2^18", [1 << 18] * 4), ("C2 64x2^24", [1 << 24] * 64)):
    pipe = MapReducePipeline(lens, world=world, rank=rank, plant_max=False)
    for _ in range(3):
        pipe.step()
    us = per_step(pipe, 50 if "tiny" in name else 20)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        pipe.graph_step(5)
        torch.cuda.synchronize()
    kern = [ev for ev in prof.key_averages() if "pass1" in ev.key]
    kus = (getattr(kern[0], "device_time_total", 0) / kern[0].count) if kern else float("nan")
    t = torch.tensor([us, kus], device="cuda")
    allv = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(allv, t)
    if rank == 0:
        print(name, "step us per rank:", [round(float(v[0]), 1) for v in allv], "kernel us:",
              [round(float(v[1]), 1) for v in allv], flush=True)
    pipe.close()
dist.destroy_process_group()

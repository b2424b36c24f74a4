"""Cost of the sharded stage-2 exchange alone (ucg_reduce_cl_xchg_f32, one
single-CTA launch per step) replayed from a CUDA graph, per rank. Dev tool."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, ".")
from paper_1505_01120_b200 import capi  # noqa: E402
from paper_1505_01120_b200.pipeline import open_exchange  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
nloc = int(sys.argv[1]) if len(sys.argv) > 1 else 16
xg = open_exchange(world, rank, nloc, rank * nloc, world * nloc)
part = torch.arange(nloc, dtype=torch.float32, device="cuda") + rank * nloc
res = torch.empty(1, device="cuda")


def call():
    capi.call("ucg_reduce_cl_xchg_f32", part.data_ptr(), nloc, 0, xg, res.data_ptr(),
              torch.cuda.current_stream().cuda_stream)


for _ in range(5):
    call()
torch.cuda.synchronize()
K = 200
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        for _ in range(K):
            call()
torch.cuda.current_stream().wait_stream(s)
g.replay()
torch.cuda.synchronize()
dist.barrier()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / K
want = float(sum(range(world * nloc)))
t = torch.tensor([us, float(res.item() == want)], device="cuda")
allv = [torch.zeros_like(t) for _ in range(world)]
dist.all_gather(allv, t)
if rank == 0:
    print(f"world {world} nloc {nloc}: exchange-only us/call per rank {[round(float(v[0]), 2) for v in allv]}, "
          f"correct {[bool(v[1]) for v in allv]}", flush=True)
dist.destroy_process_group()

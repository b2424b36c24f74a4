"""torchrun worker for tests/test_multigpu.py: a sharded C2-shaped pipeline on
N GPUs must give bit-identical partials/results to the single-GPU oracle, with
both exchanges (fused NVLink P2P in the finish kernel, and NCCL all-gather)."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_lib as O  # noqa: E402
from paper_1505_01120_b200.pipeline import MapReducePipeline, partition_sizes  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    # UCG_SHARED_GPU=1: every rank on cuda:0 (a one-GPU box). The fused
    # exchange is unchanged — IPC-mapped regions of another process, epoch-
    # tagged stores — and the ranks' kernels interleave by time slicing;
    # torch.distributed (gloo) only carries the IPC handles. NCCL cases skip
    # (NCCL refuses two ranks on one device).
    shared = os.environ.get("UCG_SHARED_GPU") == "1"
    dev = 0 if shared else int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(dev)
    if shared:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    report = {"rank": rank, "ok": True, "cases": [], "shared_gpu": shared}
    for (P, total, op, fused, exchange) in [(8, 1 << 20, "sum", True, "p2p"), (7, 300001, "max", True, "p2p"),
                                            (64, 1 << 22, "sum", False, "p2p"), (5, 100000, "sum", True, "nccl"),
                                            (3, 50000, "max", False, "nccl")]:
        if shared and exchange == "nccl":
            continue
        lens = partition_sizes(total, P)
        pipe = MapReducePipeline(lens, op=op, fused=fused, world=world, rank=rank, exchange=exchange)
        for _ in range(3):  # repeated steps exercise the epoch flags
            r = float(pipe.step().item())
        partials = [O.tree_reduce(O.map_affine(O.fill_uniform(1000 + p, lens[p]), 2.0, 1.0)
                                  if not (p == P // 2) else _planted(p, lens[p]), op) for p in range(P)]
        want = O.tree_reduce(np.array(partials, np.float32), op)
        got_local = pipe.partials.cpu().numpy()[:len(pipe.local_lens)]
        ok_local = [O.f32_bits(got_local[k]) == O.f32_bits(partials[p]) for k, p in enumerate(pipe.owned)]
        ok = all(ok_local) and O.f32_bits(np.float32(r)) == O.f32_bits(want) and pipe.exchange_error() == 0
        report["cases"].append({"P": P, "op": op, "exchange": exchange, "ok": ok, "got": r, "want": float(want)})
        report["ok"] &= ok
        pipe.close()
    # the e2e path: per-chunk uploads + launches, then the stage-2 exchange
    # alone (ucg_reduce_cl_xchg_f32) — p2p — or the NCCL all-gather
    for (P, total, op, exchange) in [(16, 1 << 22, "sum", "p2p"), (7, 300001, "max", "p2p"),
                                     (16, 1 << 22, "sum", "nccl")]:
        if shared and exchange == "nccl":
            continue
        lens = partition_sizes(total, P)
        pipe = MapReducePipeline(lens, op=op, fused=True, world=world, rank=rank, exchange=exchange)
        partials = [O.tree_reduce(O.map_affine(O.fill_uniform(1000 + p, lens[p]), 2.0, 1.0)
                                  if not (p == P // 2) else _planted(p, lens[p]), op) for p in range(P)]
        want = O.tree_reduce(np.array(partials, np.float32), op)
        pipe.setup_host_input(chunks=3)
        ok = True
        for _ in range(3):
            r = pipe.step_from_host()
            ok &= O.f32_bits(np.float32(r)) == O.f32_bits(want)
        ok &= pipe.exchange_error() == 0
        report["cases"].append({"P": P, "op": op, "exchange": exchange + "-e2e", "ok": ok, "got": r,
                                "want": float(want)})
        report["ok"] &= ok
        pipe.close()
    # sharded steps replayed from CUDA graphs (the exchange epoch advances on
    # the device): a multi-finisher table and a single-finisher one, the
    # result poisoned between replays
    for (P, total, op) in [(16, 1 << 22, "sum"), (8, 1 << 20, "max")]:
        lens = partition_sizes(total, P)
        pipe = MapReducePipeline(lens, op=op, fused=True, world=world, rank=rank, exchange="p2p")
        partials = [O.tree_reduce(O.map_affine(O.fill_uniform(1000 + p, lens[p]), 2.0, 1.0)
                                  if not (p == P // 2) else _planted(p, lens[p]), op) for p in range(P)]
        want = O.tree_reduce(np.array(partials, np.float32), op)
        ok = True
        for _ in range(3):
            pipe.result.fill_(float("nan"))
            r = float(pipe.graph_step(7).item())
            ok &= O.f32_bits(np.float32(r)) == O.f32_bits(want)
        ok &= pipe.exchange_error() == 0
        report["cases"].append({"P": P, "op": op, "exchange": "p2p-graph", "ok": ok, "got": r, "want": float(want)})
        report["ok"] &= ok
        pipe.close()
    # long chains of repeated steps (early-stream mode: each step launches
    # its successor at its first instruction; parity start tickets): eager
    # chains and graph replays at the 8-GPU shard geometry (8 partitions per
    # rank) and a single-finisher table — a ticket drawn out of order would
    # stall a rank until the 30 s trap
    chains = [(8 * world, (1 << 21) * world, "sum", 300, 60), (4, 1 << 20, "max", 600, 100)]
    if shared:  # every exchange waits for the other rank's time slice
        chains = [(8 * world, (1 << 21) * world, "sum", 20, 8), (4, 1 << 20, "max", 30, 10)]
    for (P, total, op, eager, graph) in chains:
        lens = partition_sizes(total, P)
        pipe = MapReducePipeline(lens, op=op, fused=True, world=world, rank=rank, exchange="p2p")
        partials = [O.tree_reduce(O.map_affine(O.fill_uniform(1000 + p, lens[p]), 2.0, 1.0)
                                  if not (p == P // 2) else _planted(p, lens[p]), op) for p in range(P)]
        want = O.tree_reduce(np.array(partials, np.float32), op)
        for _ in range(eager):
            pipe.step()
        ok = O.f32_bits(np.float32(pipe.result.item())) == O.f32_bits(want)
        for _ in range(4):
            pipe.result.fill_(float("nan"))
            ok &= O.f32_bits(np.float32(pipe.graph_step(graph).item())) == O.f32_bits(want)
        ok &= pipe.exchange_error() == 0
        report["cases"].append({"P": P, "op": op, "exchange": "p2p-chains", "ok": ok, "want": float(want)})
        report["ok"] &= ok
        pipe.close()
    # C3 sharded: map_cl(pi) + reduce_cl(isum2), the rank totals exchanged
    # inside the counting kernel over NVLink; T = world - 1 leaves one rank
    # without tasks (it still joins the exchange)
    from paper_1505_01120_b200 import ops
    from paper_1505_01120_b200.pipeline import open_exchange, shard_range

    xg = open_exchange(world, rank, 2, 2 * rank, 2 * world)
    for T, S in [(13, 300001), (max(1, world - 1), 70000)]:
        mine = list(shard_range(T, world, rank))
        seeds = [42 + t for t in mine]
        samples = [S + 1000 * t for t in mine]
        hits = torch.zeros(max(1, len(mine)), dtype=torch.int64, device="cuda")
        total = torch.empty(1, dtype=torch.int64, device="cuda")
        for _ in range(3):  # repeated launches exercise the epoch flags
            ops.pi_hits(seeds, samples, hits, total_out=total, xchg=xg)
        want = sum(O.pi_hits(42 + t, S + 1000 * t) for t in range(T))
        got = int(total.item())
        ok = got == want and hits.cpu().tolist()[:len(mine)] == [O.pi_hits(42 + t, S + 1000 * t) for t in mine]
        report["cases"].append({"pi_tasks": T, "ok": ok, "got": got, "want": want})
        report["ok"] &= ok
    # one write(2) per report: ranks share the stdout pipe, and print() may
    # split text and newline into two writes that other ranks interleave
    os.write(1, ("MULTIGPU " + json.dumps(report) + "\n").encode())
    dist.destroy_process_group()
    return 0 if report["ok"] else 1


def _planted(p, n):
    x = O.fill_uniform(1000 + p, n)
    x[n // 3] = 1.5
    return O.map_affine(x, 2.0, 1.0)


if __name__ == "__main__":
    sys.exit(main())

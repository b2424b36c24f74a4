"""CPU, world_size 2 over gloo: the multi-GPU host logic of the sharded
reduce_cl — partition blocks per rank (partition p -> rank floor(p*G/P)),
the padded all-gather of partials, and the reference stage-2 tree over the
gathered partials — gives exactly the single-rank result. The per-partition
partials come from the oracle here (the checker standing in for the device)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_lib as O
from paper_1505_01120_b200.pipeline import gather_index, gather_partials, partition_sizes, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    for (P, L, op) in cases:
        lens = partition_sizes(L * P + 3, P)  # ragged partitions
        mine = shard_range(P, world, rank)
        local = torch.tensor([float(O.tree_reduce(O.map_affine(O.fill_uniform(1000 + p, lens[p]), 2.0, 1.0), op))
                              for p in mine], dtype=torch.float32)
        allp = gather_partials(local, P, world)
        out.append(allp.numpy().copy())
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_combine_matches_single_rank(world):
    cases = [(64, 512, "sum"), (7, 300, "max"), (3, 100, "sum"), (1, 50, "sum")]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for i, (P, L, op) in enumerate(cases):
        lens = partition_sizes(L * P + 3, P)
        want = np.array([O.tree_reduce(O.map_affine(O.fill_uniform(1000 + p, lens[p]), 2.0, 1.0), op)
                         for p in range(P)], np.float32)
        for r in range(world):
            assert np.array_equal(res[r][i].view(np.uint32), want.view(np.uint32))
        total = O.tree_reduce(res[0][i], op)
        assert O.f32_bits(total) == O.f32_bits(O.tree_reduce(want, op))


def test_shard_ranges_cover_in_order():
    for P in (1, 3, 7, 64, 65):
        for G in (1, 2, 3, 4, 8):
            got = [p for r in range(G) for p in shard_range(P, G, r)]
            assert got == list(range(P))
            # partition p lives on rank floor(p*G/P)-ish contiguous blocks
            max_local, idx = gather_index(P, G)
            assert len(idx) == P and len(set(idx)) == P and max(idx) < G * max_local

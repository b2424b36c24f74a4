"""CPU, world_size 8 over gloo: the 8-rank sharded reduce_cl, with the
device-side peer exchange mirrored in Python.

Per rank g of G (paper_1505_01120_b200/pipeline.py shard_range): partitions
[gP/G, (g+1)P/G). The exchange region of every rank (csrc/ucg_runtime.cu
ucg_xchg_create) holds 2 parity buffers of P 64-bit slots, then P gathered
floats, then the flags at flags_offset = ceil(20P / 256) * 256. In exchange
number e (1, 2, ...), the finisher that computes partition value j of rank g
stores (e << 32 | bits(value)) into slot (e & 1) * P + part_offset_g + j of
EVERY rank's region (csrc/ucg_reduce.cu send_value); the receiver waits until
all P slots of parity buffer (e & 1) carry epoch e, then runs the reference
stage-2 tree over them in partition order (stage2). The mirror checks:

  * geometry: shards tile [0, P) in order; slot ranges of different ranks
    are disjoint and cover each parity buffer exactly; flags lie past the
    gathered floats and inside the region;
  * epoch / parity: a rank one exchange AHEAD of a peer (skew of 1) writes
    only the other parity buffer, so the peer's pending exchange still sees
    complete epoch-e slots and never a mix; the values every rank reads are
    the partials of exactly one exchange;
  * the result: every rank's stage-2 tree over the received values equals the
    single-rank reference result bit for bit (partials from the oracle).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_lib as O
from paper_1505_01120_b200.pipeline import gather_partials, partition_sizes, shard_range

WORLD = 8


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def region_geometry(p_total: int, world: int) -> dict:
    flags_offset = (20 * p_total + 255) // 256 * 256
    return {"slots_bytes": 16 * p_total, "gathered_offset": 16 * p_total, "gathered_bytes": 4 * p_total,
            "flags_offset": flags_offset, "flags_bytes": 4 * world, "region_bytes": flags_offset + 256}


def slot(epoch: int, p_total: int, part_offset: int, j: int) -> int:
    return (epoch & 1) * p_total + part_offset + j


def pack(epoch: int, v: np.float32) -> int:
    return (epoch << 32) | int(np.array([v], np.float32).view(np.uint32)[0])


def partials_for(P: int, L: int, op: str, step: int) -> np.ndarray:
    """Partition values of exchange `step` (a different input per step, so a
    mix of two exchanges would be detected)."""
    lens = partition_sizes(L * P + 3, P)
    return np.array([O.tree_reduce(O.map_affine(O.fill_uniform(1000 + 7 * step + p, lens[p]), 2.0, 1.0), op)
                     for p in range(P)], np.float32)


def _worker(rank, world, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    for (P, L, op) in cases:
        mine = shard_range(P, world, rank)
        # 1) the NCCL-path host logic (padded all-gather) at world 8
        local = torch.from_numpy(partials_for(P, L, op, 0)[mine.start:mine.stop].copy())
        allp = gather_partials(local, P, world).numpy().copy()
        # 2) the P2P exchange mirrored: each rank's region is a Python array of
        #    2P slots; "stores into peer regions" are all-to-all messages of
        #    (slot, packed) pairs. Rank 0 runs one exchange ahead (skew 1):
        #    its exchange e+1 lands before the others' exchange e is read.
        region = np.zeros(2 * P, dtype=np.uint64)
        results = []
        for e in (1, 2, 3):
            vals = partials_for(P, L, op, e)
            sends = [(slot(e, P, mine.start, j), pack(e, vals[p])) for j, p in enumerate(mine)]
            gathered = [None] * world
            dist.all_gather_object(gathered, sends)
            for r in range(world):
                for (s, v) in gathered[r]:
                    region[s] = v
            if rank != 0 or e == 1:
                # the skewed rank's next exchange (e+1) is already in flight
                ahead = partials_for(P, L, op, e + 1)
                src = [(slot(e + 1, P, shard_range(P, world, 0).start, j), pack(e + 1, ahead[p]))
                       for j, p in enumerate(shard_range(P, world, 0))] if e < 3 else []
                for (s, v) in src:
                    region[s] = v
            buf = region[(e & 1) * P:(e & 1) * P + P]
            epochs = (buf >> np.uint64(32)).astype(np.int64)
            complete = bool(np.all(epochs == e))
            got = (buf & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.float32)
            results.append((complete, got.copy(), np.float32(O.tree_reduce(got, op))))
        out.append((allp, results))
    q.put((rank, out))
    dist.destroy_process_group()


def test_geometry_world8():
    for P in (64, 67, 5, 1):
        geo = region_geometry(P, WORLD)
        assert geo["gathered_offset"] + geo["gathered_bytes"] <= geo["flags_offset"]
        assert geo["flags_offset"] + geo["flags_bytes"] <= geo["region_bytes"]
        assert geo["flags_offset"] % 256 == 0
        for e in (1, 2):
            cover = []
            for r in range(WORLD):
                rng = shard_range(P, WORLD, r)
                cover += [slot(e, P, rng.start, j) for j in range(len(rng))]
            base = (e & 1) * P
            assert sorted(cover) == list(range(base, base + P)), (P, e)
        got = [p for r in range(WORLD) for p in shard_range(P, WORLD, r)]
        assert got == list(range(P))


@pytest.mark.parametrize("cases", [[(64, 256, "sum"), (67, 100, "max"), (5, 300, "sum")]])
def test_world8_exchange_mirror(cases):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, cases, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for i, (P, L, op) in enumerate(cases):
        want0 = partials_for(P, L, op, 0)
        for r in range(WORLD):
            allp, results = res[r][i]
            assert np.array_equal(allp.view(np.uint32), want0.view(np.uint32)), (P, r)
            for k, (complete, got, total) in enumerate(results):
                e = k + 1
                want = partials_for(P, L, op, e)
                assert complete, (P, r, e)
                assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (P, r, e)
                assert O.f32_bits(total) == O.f32_bits(O.tree_reduce(want, op))

"""Device-resident mapCL -> mapCLPartition -> reduceCL pipeline over a sharded
collection (BASELINE configs 1 and 2).

Reference semantics (ucores/engine.hpp):
  y  = map_cl(x, "axpb")               :54-85   one task per element
  ps = map_cl_partition(y, "psum")     :89-114  one task per partition (concat)
  r  = reduce_cl(ps, "sum2")           :121-192 stage 2 tree over P partials

Layout in HBM: every partition's concatenated payload is one segment starting
at a 256-byte aligned float offset of one buffer (x and y share the layout).
Sharding: rank g of G holds partitions [gP/G, (g+1)P/G);
the only exchange is of the per-partition partials, after which every rank
runs the reference stage-2 tree over all P partials in partition order —
bit-identical to one GPU. Default exchange "p2p": the reduction kernel's
tail stores this rank's partials into every peer's buffer over NVLink (CUDA
IPC mapped) and waits on epoch flags, so a step is ONE launch with no
collective; "nccl" uses torch.distributed all-gather + a tree launch.

With fused=True the map and the partition reduction run as ONE kernel (read
x, write y, reduce y: 8 B/elem instead of 12); y is still materialised, so
the outputs are identical to the unfused chain.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import capi, ops

ALIGN_FLOATS = 64  # 256-byte segment alignment


def partition_sizes(n: int, num_partitions: int) -> list[int]:
    """create_dataset ceiling-first sizes (ucores/dataset.hpp:64-82)."""
    if num_partitions < 1:
        from .errors import InvalidPartitionCount

        raise InvalidPartitionCount(f"num_partitions must be >= 1, got {num_partitions}")
    base, extra = divmod(n, num_partitions)
    return [base + (1 if p < extra else 0) for p in range(num_partitions)]


def shard_range(num_partitions: int, world: int, rank: int) -> range:
    """Contiguous block of partitions owned by `rank` (partition p -> GPU floor(p*G/P))."""
    lo = (rank * num_partitions) // world
    hi = ((rank + 1) * num_partitions) // world
    return range(lo, hi)


def gather_index(num_partitions: int, world: int) -> tuple[int, list[int]]:
    """Padded all-gather layout: each rank sends max_local slots; returns
    (max_local, positions of partitions 0..P-1 in the gathered buffer)."""
    max_local = max(len(shard_range(num_partitions, world, r)) for r in range(world))
    idx = []
    for r in range(world):
        idx.extend(r * max(1, max_local) + k for k in range(len(shard_range(num_partitions, world, r))))
    return max(1, max_local), idx


def gather_partials(local, num_partitions: int, world: int, group=None, send_buf=None, gather_buf=None,
                    index=None, out=None):
    """The exchange step of a sharded reduce_cl: every rank contributes the
    partials of its partition block and receives all P partials in partition
    order (NCCL all-gather on GPUs, any torch.distributed backend works)."""
    import torch.distributed as dist

    max_local, idx = gather_index(num_partitions, world)
    dev = local.device
    if send_buf is None:
        send_buf = torch.empty(max_local, dtype=local.dtype, device=dev)
    if gather_buf is None:
        gather_buf = torch.empty(world * max_local, dtype=local.dtype, device=dev)
    if index is None:
        index = torch.tensor(idx, dtype=torch.int64, device=dev)
    if out is None:
        out = torch.empty(num_partitions, dtype=local.dtype, device=dev)
    n = local.numel()
    send_buf.fill_(0)
    if n:
        send_buf[:n].copy_(local)
    dist.all_gather_into_tensor(gather_buf, send_buf, group=group)
    torch.index_select(gather_buf, 0, index, out=out)
    return out


@dataclass
class Layout:
    """Segment layout of a set of partitions in one device buffer."""

    lens: list[int]
    begins: list[int]
    total: int

    @classmethod
    def of(cls, lens: list[int], align: int = ALIGN_FLOATS) -> "Layout":
        begins, off = [], 0
        for n in lens:
            begins.append(off)
            off += (n + align - 1) // align * align
        return cls(list(lens), begins, max(off, align))


def open_exchange(world: int, rank: int, nloc: int, part_offset: int, p_total: int, group=None) -> int:
    """A peer-exchange context (include/ucores_cuda.h ucg_xchg_*): this rank's
    IPC-exported region, every rank's handle all-gathered once through
    torch.distributed (the only host-side collective; the per-step exchange
    runs inside the kernels over NVLink) and opened. Returns the handle."""
    import ctypes as C

    import torch.distributed as dist

    h = C.c_void_p()
    capi.call("ucg_xchg_create", world, rank, nloc, part_offset, p_total, C.byref(h), phase="map_parameters")
    nbytes = int(capi.load().ucg_xchg_handle_bytes())
    mine = (C.c_char * nbytes)()
    capi.call("ucg_xchg_export", h.value, mine)
    handles = [None] * world
    dist.all_gather_object(handles, bytes(mine), group=group)
    allh = (C.c_char * (nbytes * world)).from_buffer_copy(b"".join(handles))
    capi.call("ucg_xchg_open", h.value, allh)
    return h.value


class MapReducePipeline:
    """One rank's share of the C1/C2 pipeline, inputs resident in HBM."""

    def __init__(self, part_lens: list[int], a: float = 2.0, b: float = 1.0, op: str = "sum",
                 fused: bool = True, world: int = 1, rank: int = 0, device: torch.device | None = None,
                 seed_base: int = 1000, plant_max: bool = True, group=None, exchange: str = "p2p"):
        """exchange: how a sharded reduce_cl combines partials — "p2p" (the
        reduction kernel's tail stores into peers' buffers over NVLink and
        waits on epoch flags; no collective launch) or "nccl" (all-gather +
        tree)."""
        self.P = len(part_lens)
        self.exchange = exchange
        self.part_lens = list(part_lens)
        self.a, self.b, self.op, self.fused = float(a), float(b), op, fused
        self.world, self.rank, self.group = world, rank, group
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.owned = shard_range(self.P, world, rank)
        self.local_lens = [self.part_lens[p] for p in self.owned]
        self.layout = Layout.of(self.local_lens)
        self.elements = sum(self.part_lens)
        self.local_elements = sum(self.local_lens)
        dev = self.device
        self.x = torch.empty(self.layout.total, dtype=torch.float32, device=dev)
        self.y = torch.empty_like(self.x)
        self.segtab = capi.SegTab(self.layout.begins, self.local_lens)
        self.scratch = torch.empty(max(1, self.segtab.scratch_floats), dtype=torch.float32, device=dev)
        self.partials = torch.empty(max(1, len(self.local_lens)), dtype=torch.float32, device=dev)
        self.max_local, idx = gather_index(self.P, world)
        self.gather_buf = torch.empty(world * self.max_local, dtype=torch.float32, device=dev)
        self.send_buf = torch.empty(self.max_local, dtype=torch.float32, device=dev)
        self.gather_index = torch.tensor(idx, dtype=torch.int64, device=dev)
        self.all_partials = torch.empty(max(1, self.P), dtype=torch.float32, device=dev)
        self.result = torch.empty(1, dtype=torch.float32, device=dev)
        self.seed_base = seed_base
        self.plant_max = plant_max
        self.fill()

    # -- synthetic input: partition p ~ U[0,1) from seed seed_base+p --------------
    def fill(self) -> None:
        for k, p in enumerate(self.owned):
            n = self.local_lens[k]
            if n:
                seg = self.x[self.layout.begins[k]: self.layout.begins[k] + n]
                ops.fill_uniform_(seg, self.seed_base + p)
                if self.plant_max and p == self.P // 2:
                    seg[n // 3] = 1.5  # the unique planted maximum

    def host_input(self) -> list:
        """This rank's partitions as host arrays (for oracle checks)."""
        out = []
        for k in range(len(self.local_lens)):
            b, n = self.layout.begins[k], self.local_lens[k]
            out.append(self.x[b:b + n].cpu().numpy())
        return out

    def local_output(self, k: int) -> torch.Tensor:
        b = self.layout.begins[k]
        return self.y[b:b + self.local_lens[k]]

    # -- one step ---------------------------------------------------------------
    def map_and_partials(self, stream=None) -> None:
        if self.fused:
            ops.map_affine_segment_reduce(self.x, self.y, self.segtab, self.a, self.b, self.op, self.scratch,
                                          self.partials, stream=stream)
        else:
            ops.map_affine(self.x, self.y, self.a, self.b, stream=stream)
            ops.segment_reduce(self.y, self.segtab, self.op, self.scratch, self.partials, stream=stream)

    def combine(self, stream=None) -> torch.Tensor:
        """reduce_cl stage 2 over all P partials (exchange first when sharded)."""
        if self.world == 1:
            ops.tree_reduce(self.partials, self.P, self.op, self.result, stream=stream)
            return self.result
        n = len(self.local_lens)
        if self.exchange == "p2p":
            # the fused NVLink exchange + stage-2 tree in one single-CTA launch
            if getattr(self, "xchg", None) is None:
                self._setup_xchg()
            capi.call("ucg_reduce_cl_xchg_f32", self.partials.data_ptr(), n, capi.OPS[self.op], self.xchg,
                      self.result.data_ptr(), capi.stream_handle(stream))
            return self.result
        if self.P % self.world == 0:
            # equal blocks: the gathered buffer is already in partition order
            import torch.distributed as dist

            dist.all_gather_into_tensor(self.all_partials, self.partials[:n], group=self.group)
        else:
            gather_partials(self.partials[:n], self.P, self.world, self.group, self.send_buf, self.gather_buf,
                            self.gather_index, self.all_partials)
        ops.tree_reduce(self.all_partials, self.P, self.op, self.result, stream=stream)
        return self.result

    def _setup_xchg(self) -> None:
        self.xchg = open_exchange(self.world, self.rank, len(self.local_lens), self.owned.start, self.P, self.group)

    def step(self) -> torch.Tensor:
        """One pass: map + partition reduce + reduce_cl (+ exchange when sharded)."""
        if self.world > 1 and self.exchange == "nccl":
            self.map_and_partials()
            return self.combine()
        if self.world > 1 and getattr(self, "xchg", None) is None:
            self._setup_xchg()
        xg = getattr(self, "xchg", None) if self.world > 1 else None
        if self.fused:
            ops.segment_reduce_cl(self.x, self.y, self.segtab, self.a, self.b, self.op, self.scratch, self.partials,
                                  xg, self.result)
        else:
            ops.map_affine(self.x, self.y, self.a, self.b)
            ops.segment_reduce_cl(self.y, None, self.segtab, self.a, self.b, self.op, self.scratch, self.partials,
                                  xg, self.result)
        return self.result

    def graph_step(self, steps: int = 1) -> torch.Tensor:
        """`steps` consecutive step()s replayed from one CUDA graph captured on
        first use (one GPU): the kernel nodes and their launch attributes are
        fixed, so a replay costs one cudaGraphLaunch instead of `steps`
        Python/ctypes launches, and consecutive small-table steps overlap
        launch and tail (programmatic dependent launch edges). Every step
        still runs in full: one kernel node per step. Sharded pipelines with
        the fused NVLink exchange replay too (its epoch advances on the
        device, once per exchange); every rank must replay the same count."""
        if self.world > 1 and self.exchange == "nccl":
            for _ in range(steps):
                r = self.step()
            return r
        graphs = self.__dict__.setdefault("_graphs", {})
        if steps not in graphs:
            self.step()  # warm: allocations and lazy library state outside the capture
            torch.cuda.synchronize()
            side = torch.cuda.Stream(device=self.device)
            side.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(side):
                with torch.cuda.graph(g, stream=side):
                    for _ in range(steps):
                        self.step()
            torch.cuda.current_stream().wait_stream(side)
            graphs[steps] = g
        self._poll_exchange()  # replays bypass the C entry point's error guard
        graphs[steps].replay()
        return self.result

    def _poll_exchange(self) -> None:
        """Raise PeerExchangeError if an earlier exchange timed out (reads the
        host-mapped error word: no device sync)."""
        import ctypes as C

        if getattr(self, "xchg", None) is None:
            return
        e = C.c_int(0)
        capi.call("ucg_xchg_poll", self.xchg, C.byref(e))
        if e.value:
            capi.check(capi.ERR_PEER, "run")

    def reset_exchange(self) -> None:
        """Recovery after PeerExchangeError: every rank calls this (it
        barriers on the process group) — error word, epoch and region cleared."""
        import torch.distributed as dist

        if getattr(self, "xchg", None) is None:
            return
        dist.barrier(group=self.group)
        capi.call("ucg_xchg_reset", self.xchg)
        dist.barrier(group=self.group)

    def exchange_error(self) -> int:
        """1 if a peer never published its partials (checked synchronously)."""
        import ctypes as C

        if getattr(self, "xchg", None) is None:
            return 0
        e = C.c_int(0)
        capi.call("ucg_xchg_error", self.xchg, C.byref(e))
        return e.value

    # -- end to end: inputs from pinned host memory, result back to the host ------
    def setup_host_input(self, chunks: int = 8) -> None:
        """Pinned host copy of this rank's input + per-chunk segment tables so
        the upload of chunk c+1 (copy stream) overlaps the kernel on chunk c."""
        self.host_x = torch.empty(self.layout.total, dtype=torch.float32, pin_memory=True)
        self.host_x.copy_(self.x)
        self.host_result = torch.empty(1, dtype=torch.float32, pin_memory=True)
        self.copy_stream = torch.cuda.Stream(device=self.device)
        nloc = len(self.local_lens)
        chunks = max(1, min(chunks, nloc))
        self.groups = []
        for c in range(chunks):
            k0, k1 = (c * nloc) // chunks, ((c + 1) * nloc) // chunks
            if k0 == k1:
                continue
            xb = self.layout.begins[k0]
            xe = self.layout.begins[k1 - 1] + (self.local_lens[k1 - 1] + ALIGN_FLOATS - 1) // ALIGN_FLOATS * ALIGN_FLOATS
            tab = capi.SegTab([self.layout.begins[k] - xb for k in range(k0, k1)], self.local_lens[k0:k1])
            scratch = torch.empty(max(1, tab.scratch_floats), dtype=torch.float32, device=self.device)
            self.groups.append((k0, k1, xb, xe, tab, scratch))
        self.h2d_bytes = sum((xe - xb) * 4 for (_, _, xb, xe, _, _) in self.groups)

    def step_from_host(self) -> float:
        """One end-to-end step: H2D of the shard, map+reduce, combine, D2H of the result."""
        cur = torch.cuda.current_stream(self.device)
        self.copy_stream.wait_stream(cur)  # previous step finished reading x
        for (k0, k1, xb, xe, tab, scratch) in self.groups:
            with torch.cuda.stream(self.copy_stream):
                self.x[xb:xe].copy_(self.host_x[xb:xe], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.copy_stream)
            cur.wait_event(ev)
            if self.fused:
                ops.map_affine_segment_reduce(self.x[xb:], self.y[xb:], tab, self.a, self.b, self.op, scratch,
                                              self.partials[k0:])
            else:
                ops.map_affine(self.x[xb:xe], self.y[xb:xe], self.a, self.b)
                ops.segment_reduce(self.y[xb:], tab, self.op, scratch, self.partials[k0:])
        r = self.combine()
        self.host_result.copy_(r, non_blocking=True)
        cur.synchronize()
        return float(self.host_result[0])

    def close(self) -> None:
        if getattr(self, "xchg", None):
            capi.load().ucg_xchg_destroy(self.xchg)
            self.xchg = None
        self.segtab.close()
        for g in getattr(self, "groups", []):
            g[4].close()

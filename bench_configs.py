"""The other BASELINE.json configs, measured with the same contract as
bench.py (imported by `bench.py --workload c1|c3|c4|c5`):

  c1  mapCL axpb over a 2^20-element collection in 4 partitions, then
      mapCLPartition psum + reduceCL sum2 (the CPU-runnable case)
  c3  Monte-Carlo pi via mapCL, 2^34 samples in 64 tasks (exact counts)
  c4  mapCLPartition 3x3 Sobel on a 16384x16384 u8 image in 64 row bands
  c5  mapCL dense fp32 matmul 8192^3 per partition, 8 partitions, tcgen05
  wc  WordCount word-start flags over 1 GiB of text in 64 chunks (§8(f)4)

Units (tasks / bands / partitions) are split over the ranks in contiguous
blocks; value = all units / max-over-ranks device time. The reference CPU
path (oracle/_ref/ref_harness bench-workload) is timed on a bounded sample.
"""
from __future__ import annotations

import json
import os
import statistics
import subprocess
import time

import torch

import bench as B
from paper_1505_01120_b200 import capi, ops
from paper_1505_01120_b200.pipeline import MapReducePipeline, shard_range

CONFIGS = json.loads((B.ROOT / "BASELINE.json").read_text())["configs"]


def _timed(fn, k, barrier):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    barrier()
    return e0.elapsed_time(e1) / k


def _soak(fn, warmup, barrier, seconds=1.0):
    """Inside the clock sampler, before a timed region: W warm-up calls, then
    ~1 s of untimed calls, so nvidia-smi is up and sampling (its start-up
    no longer overlaps a few-ms timed region) and the clocks are at steady
    state — as bench.py's C2 arm does."""
    for _ in range(max(3, warmup)):
        fn()
    barrier()
    end = time.perf_counter() + seconds
    while time.perf_counter() < end:
        for _ in range(10):
            fn()
        torch.cuda.synchronize()
    barrier()


class _Duplex:
    """One end-to-end step in pieces: piece i's upload (copy-in stream), its
    kernel (the current stream) and its download (copy-out stream), so the
    uploads of later pieces overlap the downloads of earlier ones on the two
    copy engines (PCIe is full duplex). Every step still moves all of its
    inputs up and all of its outputs down."""

    def __init__(self, dev):
        self.s_in = torch.cuda.Stream(device=dev)
        self.s_out = torch.cuda.Stream(device=dev)

    def step(self, npieces, h2d, run, d2h):
        cur = torch.cuda.current_stream()
        self.s_in.wait_stream(cur)
        ups = []
        with torch.cuda.stream(self.s_in):
            for i in range(npieces):
                h2d(i)
                e = torch.cuda.Event()
                e.record(self.s_in)
                ups.append(e)
        for i in range(npieces):
            cur.wait_event(ups[i])
            run(i)
            e = torch.cuda.Event()
            e.record(cur)
            self.s_out.wait_event(e)
            with torch.cuda.stream(self.s_out):
                d2h(i)
        cur.wait_stream(self.s_out)
        cur.synchronize()


def _max_over_ranks(vals, world, dev):
    if world == 1:
        return vals
    import torch.distributed as dist

    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t]


def _ref_workload(argv, timeout=900):
    out = subprocess.run([str(B.REF_HARNESS), "bench-workload"] + argv + ["--threads", str(os.cpu_count() or 1)],
                         check=True, capture_output=True, text=True, timeout=timeout).stdout
    return json.loads(out.strip().splitlines()[-1])


def _traffic(key: str, share: float):
    """ncu DRAM bytes of one full-size launch (profiles/ncu_summary.json),
    scaled to this rank's share of the units; None when not captured."""
    v = B.load_traffic(key)
    return None if v is None else int(v * share)


def _line(args, world, workload, metric_desc, value, unit, step_ms, launches, clk, e2e, roofline, cpu, config):
    return {"metric": f"{B.METRIC} [{workload}: {metric_desc}]", "value": value, "unit": unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": config.pop("dtype"), "data": "synthetic",
            "config": config, "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "gpu_launches": launches,
            "clocks": clk.summary()}


def run(args, world, rank, local):
    dev = torch.device("cuda", local)
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize()

    capi.load()
    peak_hbm, peak_kind = B.load_peak()
    k, w = args.steps, max(3, args.warmup)
    cpu = None
    line = None
    if args.workload == "c1":
        # C1 is too small to shard — at N > 1 every GPU runs the
        # whole 2^20-element collection as an independent replica (weak
        # scaling: value = all replicas' elements / max-over-ranks time)
        lens = [1 << 18] * 4
        pipe = MapReducePipeline(lens, world=1, rank=0, device=dev, plant_max=False)
        for _ in range(w):
            pipe.step()
        # the K timed steps replayed from ONE CUDA graph of K one-kernel steps:
        # at 4 MiB a step is launch-latency bound; inside the graph consecutive
        # steps are joined by programmatic-dependent-launch edges, so step k+1's
        # grid ramps up during step k's single-CTA tail
        for _ in range(w):
            pipe.graph_step()
        pipe.graph_step(k)  # capture + warm replay
        with B.ClockSampler(local) as clk:
            _soak(pipe.graph_step, w, barrier)
            ms = _timed(lambda: pipe.graph_step(k), 1, barrier) / k
            launches = k  # one k_segment_pass1 node per step (graph replays bypass the C launch counter)
            kern = _timed(pipe.map_and_partials, k, barrier)
        r_graph = float(pipe.result.item())
        pipe.step()
        torch.cuda.synchronize()
        assert float(pipe.result.item()) == r_graph  # graph replay == eager step, bitwise
        # e2e chunks (UCG_C1_E2E_CHUNKS, A/B): 4 MB of x is one upload's
        # worth; per-chunk host work (copy, event, launch) costs more than the
        # overlap gains at this size
        pipe.setup_host_input(chunks=int(os.environ.get("UCG_C1_E2E_CHUNKS", "1")))
        for _ in range(2):
            pipe.step_from_host()
        e2e_ms = _timed(pipe.step_from_host, k, barrier)
        ms, kern, e2e_ms = _max_over_ranks([ms, kern, e2e_ms], world, dev)
        n = pipe.elements * world  # replicas
        if rank == 0:
            r = B.run_ref_harness(4, 1 << 18, 3, 1, "sum", os.cpu_count() or 1)
            cpu = {"value": r["elements"] / statistics.median(r["step_s"]), "unit": "elements/s",
                   "cores": os.cpu_count(), "kind": "reference", "sample": "the full C1 workload (2^20 fp32, 4 partitions)"}
        achieved = 8 * pipe.local_elements / (kern * 1e-3) / 1e9
        line = _line(args, world, "c1", CONFIGS[0], n / (ms * 1e-3), "elements/s", ms, launches, clk,
                     {"value": n / (e2e_ms * 1e-3), "unit": "elements/s", "h2d_bytes_per_step": pipe.h2d_bytes * world,
                      "d2h_bytes_per_step": 4 * world},
                     {"bound": "latency", "achieved": achieved, "peak": peak_hbm, "unit": "GB/s",
                      "frac": achieved / peak_hbm, "traffic": None, "peak_kind": peak_kind,
                      "note": "4 MiB collection: L2-resident and launch-latency bound (1 kernel per step; the K steps replayed from one CUDA graph with programmatic-dependent-launch edges); no HBM claim"},
                     cpu, {"workload": CONFIGS[0], "elements": n, "partitions": 4, "dtype": "f32", "fused": True,
                           "l2": "no flush: the 4 MiB collection is L2-resident by size (latency-bound case, not the headline)",
                           "sharding": "replicas: every GPU runs the whole collection" if world > 1 else "1 GPU"})
        if world > 1:
            line["scaling"] = "weak"
        pipe.close()
    elif args.workload == "c3":
        S, T = 1 << 34, 64
        mine = shard_range(T, world, rank)
        seeds = [42 + t for t in mine]
        samples = [S // T + (1 if t < S % T else 0) for t in mine]
        hits = torch.empty(max(1, len(seeds)), dtype=torch.int64, device=dev)
        total = torch.empty(1, dtype=torch.int64, device=dev)
        total_host = torch.empty(1, dtype=torch.int64).pin_memory()

        xg = None
        if world > 1:
            from paper_1505_01120_b200.pipeline import open_exchange

            xg = open_exchange(world, rank, 2, 2 * rank, 2 * world)

        def fn():
            # map_cl(pi) over this rank's tasks + reduce_cl(isum2) in one launch;
            # sharded: the same launch's last CTA exchanges the rank totals over
            # NVLink (P2P stores + epoch flags), so every rank ends with the sum
            ops.pi_hits(seeds, samples, hits, total_out=total, xchg=xg)
        fn()
        with B.ClockSampler(local) as clk:
            _soak(fn, args.warmup, barrier)
            l0 = capi.launch_count()
            ms = _timed(fn, k, barrier)
            launches = capi.launch_count() - l0

        def e2e():
            fn()
            total_host.copy_(total, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        e2e_ms = _timed(e2e, k, barrier)
        ms, e2e_ms = _max_over_ranks([ms, e2e_ms], world, dev)
        fn()
        total_hits = int(total.item())
        assert total_hits == int(hits.sum().item()) or world > 1
        if world > 1:  # the fused exchange's sum equals an NCCL all-reduce of the rank totals
            import torch.distributed as dist

            chk = hits.sum().reshape(1).clone()
            dist.all_reduce(chk)
            assert int(chk.item()) == total_hits, (int(chk.item()), total_hits)
        if rank == 0:
            r = _ref_workload(["--w", "pi", "--samples", str(1 << 28), "--tasks", "64", "--steps", "1", "--warmup", "0"])
            cpu = {"value": r["units"] / statistics.median(r["step_s"]), "unit": "samples/s", "cores": r["threads"],
                   "kind": "reference", "sample": "2^28 samples in 64 tasks (the C3 task shape, 1/64 of the samples)"}
        ipc_peak = 148 * 4 * (clk.summary()["sm_mhz"] or 1965.0) * 1e6 / 1e9  # warp-instr/s (G), 4 schedulers/SM
        instr_per_sample = 52.75  # SASS of the k_pi inner loop: 211 per 4 samples (ALU ~29, FMA ~17, FP64 6)
        achieved = (S / world) / (ms * 1e-3) * instr_per_sample / 32 / 1e9
        line = _line(args, world, "c3", CONFIGS[2], S / (ms * 1e-3), "samples/s", ms, launches, clk,
                     {"value": S / (e2e_ms * 1e-3), "unit": "samples/s", "h2d_bytes_per_step": 16 * T,
                      "d2h_bytes_per_step": 8 * world},
                     {"bound": "issue", "achieved": achieved, "peak": ipc_peak, "unit": "Gwarp-instr/s",
                      "frac": achieved / ipc_peak, "traffic": 0, "note": "integer-ALU / issue bound; no HBM traffic"},
                     cpu, {"workload": CONFIGS[2], "samples": S, "tasks": T, "dtype": "u64/f64->i64",
                           "hits_total": total_hits,
                           "l2": "n/a: no input data (samples generated in registers)",
                           "exchange": "none" if world == 1 else "rank totals exchanged inside the counting kernel over NVLink (P2P stores + epoch flags)"})
    elif args.workload == "c4":
        H = W = 16384
        R = 256
        nb = H // R
        mine = shard_range(nb, world, rank)
        ln = len(mine)
        inp = torch.empty(max(1, ln) * (R + 2) * W, dtype=torch.uint8, device=dev)
        ops.fill_bytes_(inp, 7)
        out = torch.empty(max(1, ln) * R * W, dtype=torch.uint8, device=dev)
        in_off = [b * (R + 2) * W for b in range(ln)]
        out_off = [b * R * W for b in range(ln)]
        fn = lambda: ops.sobel_bands(inp, in_off, out, out_off, [R] * ln, W)
        fn()
        with B.ClockSampler(local) as clk:
            _soak(fn, args.warmup, barrier)
            l0 = capi.launch_count()
            ms = _timed(fn, k, barrier)
            launches = capi.launch_count() - l0
        host_in = torch.empty_like(inp, device="cpu").pin_memory()
        host_out = torch.empty_like(out, device="cpu").pin_memory()

        host_in.copy_(inp)
        # e2e in pieces of 8 bands: uploads overlap downloads (_Duplex)
        duplex, per_piece = _Duplex(dev), 8
        npieces = (ln + per_piece - 1) // per_piece if ln else 0
        ib, ob = (R + 2) * W, R * W

        def h2d(i):
            b0, b1 = i * per_piece, min(ln, (i + 1) * per_piece)
            inp[b0 * ib:b1 * ib].copy_(host_in[b0 * ib:b1 * ib], non_blocking=True)

        def run(i):
            b0, b1 = i * per_piece, min(ln, (i + 1) * per_piece)
            ops.sobel_bands(inp, in_off[b0:b1], out, out_off[b0:b1], [R] * (b1 - b0), W)

        def d2h(i):
            b0, b1 = i * per_piece, min(ln, (i + 1) * per_piece)
            host_out[b0 * ob:b1 * ob].copy_(out[b0 * ob:b1 * ob], non_blocking=True)

        e2e = lambda: duplex.step(npieces, h2d, run, d2h)  # noqa: E731
        e2e()
        e2e_matches = bool(torch.equal(host_out, out.cpu()))
        e2e_ms = _timed(e2e, k, barrier)
        ms, e2e_ms = _max_over_ranks([ms, e2e_ms], world, dev)
        if rank == 0:
            r = _ref_workload(["--w", "sobel", "--height", "2048", "--width", str(W), "--rows", str(R), "--steps", "1",
                               "--warmup", "0"])
            cpu = {"value": r["units"] / statistics.median(r["step_s"]), "unit": "pixels/s", "cores": r["threads"],
                   "kind": "reference", "sample": "2048x16384 (8 of the 64 bands)"}
        algo = ln * ((R + 2) * W + R * W)
        achieved = algo / (ms * 1e-3) / 1e9
        line = _line(args, world, "c4", CONFIGS[3], H * W / (ms * 1e-3), "pixels/s", ms, launches, clk,
                     {"value": H * W / (e2e_ms * 1e-3), "unit": "pixels/s",
                      "h2d_bytes_per_step": nb * (R + 2) * W, "d2h_bytes_per_step": H * W,
                      "pipeline": "pieces of 8 bands: upload, kernel, download; uploads overlap downloads",
                      "matches_device_result": e2e_matches},
                     {"bound": "hbm", "achieved": achieved, "peak": peak_hbm, "unit": "GB/s",
                      "frac": achieved / peak_hbm, "traffic": _traffic("sobel_dram_bytes", ln / nb),
                      "peak_kind": peak_kind, "algorithmic_bytes_per_launch": algo},
                     cpu, {"workload": CONFIGS[3], "height": H, "width": W, "bands": nb, "rows_per_band": R,
                           "dtype": "u8", "l2": "inputs larger than L2 (257 MiB image in, 256 MiB out)"})
    elif args.workload == "c5":
        # BASELINE: "dense fp32 matrix multiply ... tensor-core path". The line's
        # value is the fp32-faithful product (ucg_gemm_f32: 3xTF32 split on the
        # tcgen05 CTA-pair kernel, k-chunks of 256 added in fp32 round-to-
        # nearest; SGEMM-level error); the plain TF32 product is reported beside
        # it ("tf32") against cuBLAS TF32.
        n, P = 8192, 8
        mine = shard_range(P, world, rank)
        A = torch.empty(n, n, device=dev)
        Bm = torch.empty(n, n, device=dev)
        Cm = torch.empty(n, n, device=dev)

        def fill():
            ops.fill_uniform_(A, 100)
            ops.fill_uniform_(Bm, 101)
            A.mul_(2).sub_(1)  # U[-1, 1)
            Bm.mul_(2).sub_(1)
        fill()
        fn32 = lambda: [ops.gemm_f32(A, Bm, Cm, n) for _ in mine]  # noqa: E731
        fntf = lambda: [ops.gemm_tf32(A, Bm, Cm, n) for _ in mine]  # noqa: E731
        fn32()
        fntf()
        with B.ClockSampler(local) as clk:
            _soak(fn32, args.warmup, barrier)
            l0 = capi.launch_count()
            ms32 = _timed(fn32, k, barrier)
            launches = capi.launch_count() - l0  # split x2 + GEMM per partition
            mstf = _timed(fntf, k, barrier)
        torch.backends.cuda.matmul.allow_tf32 = True
        for _ in range(3):  # cuBLAS handle / heuristics / workspace outside the timed region
            torch.matmul(A, Bm)
        cub = _timed(lambda: torch.matmul(A, Bm), k, barrier)
        # accuracy of both modes on 256 sampled entries against fp64
        idx = torch.randint(0, n, (256, 2), generator=torch.Generator().manual_seed(7)).tolist()
        rows = torch.tensor([i for i, _ in idx], device=dev)
        cols = torch.tensor([j for _, j in idx], device=dev)
        ref = (A[rows].double() * Bm[:, cols].t().double()).sum(1)
        rms = float(ref.pow(2).mean().sqrt())
        ops.gemm_f32(A, Bm, Cm, n)
        err32 = float((Cm[rows, cols].double() - ref).abs().max()) / rms
        ops.gemm_tf32(A, Bm, Cm, n)
        errtf = float((Cm[rows, cols].double() - ref).abs().max()) / rms
        hA = torch.empty_like(A, device="cpu").pin_memory()
        hC = torch.empty_like(Cm, device="cpu").pin_memory()
        hA.copy_(A)

        # e2e: per partition A, B up, the product, C down — double-buffered, so
        # partition i+1's upload (copy-in stream) runs under partition i's
        # GEMM and download (copy-out stream)
        Ab, Bb, Cb = [A, torch.empty_like(A)], [Bm, torch.empty_like(Bm)], [Cm, torch.empty_like(Cm)]
        s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)

        def e2e():
            cur = torch.cuda.current_stream()
            s_in.wait_stream(cur)
            kdone, ddone = {}, {}
            for i, _ in enumerate(mine):
                j = i % 2
                with torch.cuda.stream(s_in):
                    if i >= 2:
                        s_in.wait_event(kdone[i - 2])  # GEMM i-2 has read buffer j
                    Ab[j].copy_(hA, non_blocking=True)
                    Bb[j].copy_(hA, non_blocking=True)
                    up = torch.cuda.Event()
                    up.record(s_in)
                cur.wait_event(up)
                if i >= 2:
                    cur.wait_event(ddone[i - 2])  # C buffer j downloaded
                ops.gemm_f32(Ab[j], Bb[j], Cb[j], n)
                kdone[i] = torch.cuda.Event()
                kdone[i].record(cur)
                s_out.wait_event(kdone[i])
                with torch.cuda.stream(s_out):
                    hC.copy_(Cb[j], non_blocking=True)
                    ddone[i] = torch.cuda.Event()
                    ddone[i].record(s_out)
            cur.wait_stream(s_out)
            cur.synchronize()
        e2e_ms = _timed(e2e, max(1, k // 4), barrier)
        ms32, mstf, cub, e2e_ms = _max_over_ranks([ms32, mstf, cub, e2e_ms], world, dev)
        flops = 2.0 * n ** 3 * P
        if rank == 0:
            r = _ref_workload(["--w", "matmul", "--n", "256", "--parts", "2", "--steps", "1", "--warmup", "0"])
            cpu = {"value": r["units"] / statistics.median(r["step_s"]), "unit": "FLOP/s", "cores": r["threads"],
                   "kind": "reference", "sample": "2 partitions at n=256 (the fp32 class-D run(); 8192^3 is infeasible on CPU)"}
        nloc = max(1, len(mine))
        peak = 2.0 * n ** 3 / (cub * 1e-3) / 1e12  # cuBLAS TF32, TF/s
        # the fp32-faithful kernel issues three TF32 products per fp32 product
        tc32 = 3 * 2.0 * n ** 3 / (ms32 * 1e-3 / nloc) / 1e12
        tctf = 2.0 * n ** 3 / (mstf * 1e-3 / nloc) / 1e12
        line = _line(args, world, "c5", CONFIGS[4], flops / (ms32 * 1e-3), "FLOP/s", ms32, launches, clk,
                     {"value": flops / (e2e_ms * 1e-3), "unit": "FLOP/s",
                      "h2d_bytes_per_step": P * 2 * n * n * 4, "d2h_bytes_per_step": P * n * n * 4,
                      "pipeline": "double-buffered partitions: the next A, B upload under this product and its C "
                                  "download"},
                     {"bound": "tensor", "achieved": tc32, "peak": peak, "unit": "TFLOP/s", "frac": tc32 / peak,
                      "traffic": _traffic("gemm_f32_dram_bytes", 1.0), "traffic_note": "ncu DRAM bytes of one "
                      "8192^3 fp32-faithful launch (profiles/ncu_summary.json r02)",
                      "peak_kind": "cuBLAS TF32 8192^3 measured in this run",
                      "note": "achieved counts the tensor work: 3 TF32 products (Ahi*Bhi, Ahi*Blo, Alo*Bhi) per fp32 "
                              "product; the split pass (0.25 ms, HBM-bound) is inside the timed step"},
                     cpu, {"workload": CONFIGS[4], "n": n, "partitions": P,
                           "dtype": "f32 (fp32-faithful: 3xTF32 split on tcgen05, fp32 accumulate, k-chunks of 256 "
                                    "added in fp32 round-to-nearest)",
                           "max_abs_err_over_rms_256_sampled": err32,
                           "l2": "inputs larger than L2 (8 partitions x 512 MiB A||B per step)"})
        line["tf32"] = {
            "value": flops / (mstf * 1e-3), "unit": "FLOP/s", "ms_per_step": mstf, "kernel": "ucg_gemm_tf32",
            "roofline_frac": tctf / peak, "max_abs_err_over_rms_256_sampled": errtf,
            "note": "plain TF32 (the tensor core reads the top 19 bits of each fp32 operand): the same kernel with "
                    "one product per fp32 product, at cuBLAS TF32 parity"}
    elif args.workload == "c1lit":
        # the C1 literal form — 2^20 one-float elements — through
        # the reference API: the GPU drop-in driver (one batched launch per wave)
        # and the device-resident DeviceEngine, against the reference's
        # one-task-per-element host path. An API-level, end-to-end number: host
        # Elements in, one Element out, Dataset construction timed.
        from paper_1505_01120_b200 import engine_capi

        n, P = 1 << 20, 4
        xd = torch.empty(n, dtype=torch.float32, device=dev)
        ops.fill_uniform_(xd, 12345)
        xh = xd.cpu().numpy()
        runs, launches = {}, None
        if rank == 0:
            with B.ClockSampler(local) as clk:
                for mode in ("device", "batched"):
                    engine_capi.literal_f32(xh[:4096], P, mode=mode, gpus=1)  # warm: library and GPU state
                    ts, r = [], None
                    reps = max(3, min(k, 5))
                    l0 = capi.launch_count()
                    for _ in range(reps):
                        r, sec = engine_capi.literal_f32(xh, P, mode=mode, gpus=1)
                        ts.append(sec)
                    if mode == "device":
                        launches = (capi.launch_count() - l0) // reps
                    runs[mode] = (statistics.median(ts), r)
            rr = B.run_ref_harness_literal(n, P)
            ref_s = statistics.median(rr["step_s"])
            ref_bits = rr["result_bits"]
            cpu = {"value": n / ref_s, "unit": "elements/s", "cores": rr["threads"], "kind": "reference",
                   "sample": "the full literal workload: 2^20 one-float elements in 4 partitions, one map task per element"}
            sec_d, r_d = runs["device"]
            sec_b, r_b = runs["batched"]
            import numpy as np

            bits = lambda v: format(int(np.float32(v).view(np.uint32)), "08x")
            match = bits(r_d) == bits(r_b) == ref_bits
            line = _line(args, world, "c1lit", "C1 literal form: 2^20 one-float elements (SURVEY 8(f)3)",
                         n / sec_d, "elements/s", sec_d * 1e3, launches, clk,
                         {"value": n / sec_d, "unit": "elements/s", "h2d_bytes_per_step": 4 * n,
                          "d2h_bytes_per_step": 4, "note": "the value itself is end to end (host Elements in)"},
                         {"bound": "host", "achieved": None, "peak": None, "unit": None, "frac": None,
                          "traffic": None, "note": "dominated by building 2^20 host Elements (timed in every arm)"},
                         cpu, {"workload": "C1 literal: 2^20 fp32 one-float elements, 4 partitions",
                               "dtype": "f32", "path": "ucores_b200::DeviceEngine via ucd_literal_f32",
                               "seam_a_batched_elements_per_s": n / sec_b, "results_match_reference": match,
                               "result_bits": bits(r_d)})
    elif args.workload == "wc":
        # WordCount word-start flags over create_from_text chunks.
        # Every chunk ends on a delimiter (dataset.hpp:94-112), so the flags of
        # the concatenated chunks are the concatenation of per-chunk flags: one
        # launch covers all of a GPU's chunks.
        total, chunks = 1 << 30, 64
        per = total // chunks
        mine = shard_range(chunks, world, rank)
        ln = len(mine)
        text = torch.empty(max(1, ln) * per, dtype=torch.uint8, device=dev)
        ops.fill_bytes_(text, 11)
        alphabet = (b" \t\n\r" * 12 + b"abcdefghijklmnopqrstuvwxyz0123456789" * 6)[:256]
        lut = torch.tensor(list(alphabet.ljust(256, b"e")), dtype=torch.uint8, device=dev)
        step_b = 1 << 26
        for o in range(0, text.numel(), step_b):
            seg = text[o:o + step_b]
            seg.copy_(lut[seg.to(torch.int32)])
        text.view(max(1, ln), per)[:, -1] = ord("\n")  # chunk ends on a delimiter
        flags = torch.empty_like(text)
        fn = lambda: ops.word_start_flags(text, flags)
        fn()
        with B.ClockSampler(local) as clk:
            _soak(fn, args.warmup, barrier)
            l0 = capi.launch_count()
            ms = _timed(fn, k, barrier)
            launches = capi.launch_count() - l0
        host_in = torch.empty_like(text, device="cpu").pin_memory()
        host_in.copy_(text)
        host_out = torch.empty_like(flags, device="cpu").pin_memory()

        # e2e in pieces of 8 chunks (each ends on a delimiter, so a piece's
        # flags are exact on their own): uploads overlap downloads (_Duplex)
        duplex, per_piece = _Duplex(dev), 8 * per
        npieces = (text.numel() + per_piece - 1) // per_piece if ln else 0

        def h2d(i):
            text[i * per_piece:(i + 1) * per_piece].copy_(host_in[i * per_piece:(i + 1) * per_piece], non_blocking=True)

        def run(i):
            ops.word_start_flags(text[i * per_piece:(i + 1) * per_piece], flags[i * per_piece:(i + 1) * per_piece])

        def d2h(i):
            host_out[i * per_piece:(i + 1) * per_piece].copy_(flags[i * per_piece:(i + 1) * per_piece],
                                                             non_blocking=True)

        e2e = lambda: duplex.step(npieces, h2d, run, d2h)  # noqa: E731
        fn()
        want_flags = flags.cpu()
        e2e()
        e2e_matches = bool(torch.equal(host_out, want_flags))
        e2e_ms = _timed(e2e, k, barrier)
        ms, e2e_ms = _max_over_ranks([ms, e2e_ms], world, dev)
        words = int(flags.sum(dtype=torch.int64).item()) if ln else 0
        if rank == 0:
            r = _ref_workload(["--w", "wordcount", "--bytes", str(1 << 26), "--chunk", str(1 << 22), "--steps", "1",
                               "--warmup", "0"])
            cpu = {"value": r["units"] / statistics.median(r["step_s"]), "unit": "bytes/s", "cores": r["threads"],
                   "kind": "reference",
                   "sample": ("64 MiB synthetic corpus in 4 MiB create_from_text chunks, map_cl(wordcount): per-byte "
                              "word-start flags (run) + tokenised tables (map_return_value, host)")}
        algo = 2 * ln * per
        achieved = algo / (ms * 1e-3) / 1e9
        line = _line(args, world, "wc", "WordCount word-start flags over create_from_text chunks (SURVEY 8(f)4)",
                     total / (ms * 1e-3), "bytes/s", ms, launches, clk,
                     {"value": total / (e2e_ms * 1e-3), "unit": "bytes/s", "h2d_bytes_per_step": total,
                      "d2h_bytes_per_step": total, "note": "text up, flags down (the host tokeniser's input)",
                      "pipeline": "pieces of 8 chunks: upload, kernel, download; uploads overlap downloads",
                      "matches_device_result": e2e_matches},
                     {"bound": "hbm", "achieved": achieved, "peak": peak_hbm, "unit": "GB/s",
                      "frac": achieved / peak_hbm, "traffic": _traffic("wordflags_dram_bytes", ln / chunks),
                      "peak_kind": peak_kind, "algorithmic_bytes_per_launch": algo},
                     cpu, {"workload": "1 GiB synthetic text in 64 chunks of 16 MiB, word-start flags (u8 per byte)",
                           "bytes": total, "chunks": chunks, "dtype": "u8", "word_starts_this_rank": words,
                           "l2": "inputs larger than L2 (1 GiB text)"})
    if rank == 0 and line is not None:
        B.emit(line)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0

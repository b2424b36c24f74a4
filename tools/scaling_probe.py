"""Per-GPU shard sizes of the C2 strong-scaling run (64/G partitions of 2^24)
on ONE GPU: step time, and pass-1 / finish kernel durations from CUPTI
(torch.profiler, no replay), across work-item sizes. Dev tool.

    python tools/scaling_probe.py [--items 11,12,13,14] [--gs 1,2,4,8]
"""
import argparse
import json
import math
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_1505_01120_b200.pipeline import MapReducePipeline  # noqa: E402

HBM = 6434.2


def step_ms(pipe, reps=30, warm=5):
    for _ in range(warm):
        pipe.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        pipe.step()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def b2b_ms(pipe, reps=50):
    """Back-to-back steps (as bench.py times them): launch gaps included,
    launch latency hidden."""
    for _ in range(5):
        pipe.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        pipe.step()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def kernel_us(pipe, reps=10):
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            pipe.step()
        torch.cuda.synchronize()
    out = {}
    for ev in prof.key_averages():
        name = ev.key
        tag = "pass1" if "pass1" in name else "finish" if "finish" in name else None
        if tag:
            dev_us = getattr(ev, "device_time_total", None) or getattr(ev, "cuda_time_total", 0)
            out[tag] = dev_us / max(ev.count, 1)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--items", default="0,11,12,13,14")
    ap.add_argument("--gs", default="1,2,4,8")
    ap.add_argument("--op", default="sum")
    args = ap.parse_args()
    res = []
    for g in [int(v) for v in args.gs.split(",")]:
        P = 64 // g
        n = P << 24
        for L in [int(v) for v in args.items.split(",")]:
            if L:
                os.environ["UCG_ITEM_LOG2"] = str(L)
            else:
                os.environ.pop("UCG_ITEM_LOG2", None)
            pipe = MapReducePipeline([1 << 24] * P, op=args.op, fused=True)
            ms = step_ms(pipe)
            b2b = b2b_ms(pipe)
            k = kernel_us(pipe)
            rec = {"G": g, "elems": n, "item_log2": round(math.log2(n / pipe.segtab.scratch_floats), 2),
                   "variant": os.environ.get("UCG_PASS1_VARIANT", "0"),
                   "step_ms": round(ms, 4), "b2b_ms": round(b2b, 4), "frac_b2b": round(8 * n / b2b / 1e6 / HBM, 4), "frac_step": round(8 * n / ms / 1e6 / HBM, 4),
                   "pass1_us": round(k.get("pass1", 0), 1), "finish_us": round(k.get("finish", 0), 1),
                   "frac_pass1": round(8 * n / (k.get("pass1", 1) * 1e3) / HBM, 4)}
            print(json.dumps(rec), flush=True)
            res.append(rec)
            pipe.close()
            del pipe
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

"""Sharded reduce_cl on >= 2 GPUs (torchrun, one process per GPU): the fused
NVLink P2P exchange and the NCCL exchange both give the single-GPU bits.
Skipped on boxes with fewer than 2 GPUs."""
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.gpu
def test_sharded_pipeline_bit_identical():
    import torch

    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    world = n  # every visible GPU (8 on an 8-GPU box)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                        "--master-addr", "127.0.0.1", "--master-port", "29533",
                        str(ROOT / "tests" / "multigpu_worker.py")], capture_output=True, text=True, timeout=600)
    import json
    import re

    reports = [json.JSONDecoder().raw_decode(r.stdout, m.end())[0] for m in re.finditer(r"MULTIGPU ", r.stdout)]
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0, r.stderr[-3000:]
    assert sorted(d["rank"] for d in reports) == list(range(world)), r.stdout[-3000:]
    bad = [(d["rank"], c) for d in reports for c in d["cases"] if not c["ok"]]
    assert not bad, bad


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 8])
def test_sharded_ranks_one_gpu(world):
    """The sharded path at world size 2 and 8 on ONE GPU (every rank on cuda:0):
    the same IPC-mapped regions, epoch-tagged 64-bit stores and graph-
    replayed steps as across GPUs, the two processes' kernels interleaved by
    time slicing; torch.distributed (gloo) only carries the IPC handles. Every
    rank's partials and result must equal the single-GPU bits — the multi-
    rank protocol (8 ranks: the driver's 8-GPU geometry) checked on a
    one-GPU box."""
    import json
    import os
    import re

    try:
        mode = subprocess.run(["nvidia-smi", "-i", "0", "--query-gpu=compute_mode", "--format=csv,noheader"],
                              capture_output=True, text=True, timeout=60).stdout.strip()
    except Exception:
        mode = ""
    if mode and mode.lower() != "default":
        pytest.skip(f"compute mode {mode}: one context per GPU")
    env = dict(os.environ, UCG_SHARED_GPU="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                        "--master-addr", "127.0.0.1", "--master-port", str(29547 + world),
                        str(ROOT / "tests" / "multigpu_worker.py")], capture_output=True, text=True, timeout=600,
                       env=env)
    reports = [json.JSONDecoder().raw_decode(r.stdout, m.end())[0] for m in re.finditer(r"MULTIGPU ", r.stdout)]
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0, r.stderr[-3000:]
    assert sorted(d["rank"] for d in reports) == list(range(world)), r.stdout[-3000:]
    assert all(d["shared_gpu"] for d in reports)
    bad = [(d["rank"], c) for d in reports for c in d["cases"] if not c["ok"]]
    assert not bad, bad

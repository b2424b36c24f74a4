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

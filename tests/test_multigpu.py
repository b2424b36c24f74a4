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
    world = min(n, 4)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                        "--master-addr", "127.0.0.1", "--master-port", "29533",
                        str(ROOT / "tests" / "multigpu_worker.py")], capture_output=True, text=True, timeout=600)
    lines = [l for l in r.stdout.splitlines() if l.startswith("MULTIGPU ")]
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0, r.stderr[-3000:]
    assert len(lines) == world

"""CPU: bench.py's launch contract. `--gpus N` outside torchrun relaunches
itself as N ranks (rank 0 alone prints ONE JSON line on stdout); inside
torchrun WORLD_SIZE must equal --gpus. Uses the reference arm (CPU only) at a
tiny size."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "oracle" / "_ref" / "ref_harness"


@pytest.mark.skipif(not REF.exists(), reason="oracle/_ref not built")
@pytest.mark.parametrize("gpus", [1, 2])
def test_reference_arm_one_line(gpus):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", str(gpus),
                        "--parts", "4", "--part-len", "4096", "--steps", "2", "--warmup", "1"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == gpus and d["steps"] == 2 and d["warmup"] == 1
    assert d["config"]["elements"] == 4 * 4096 and d["config"]["partitions"] == 4  # the same config, not a sample
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "reference"
    assert d["steps_requested"] == 2 and d["warmup_requested"] == 1


@pytest.mark.skipif(not REF.exists(), reason="oracle/_ref not built")
def test_reference_arm_step_cap():
    """Each reference step is the whole workload on the CPU: the arm times at
    most --ref-steps of the K steps after one warm-up, and says so."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--parts", "2", "--part-len",
                        "1024", "--steps", "20", "--warmup", "5", "--ref-steps", "3"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.strip()][-1])
    assert (d["steps"], d["warmup"], d["steps_requested"], d["warmup_requested"]) == (3, 1, 20, 5)


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "3"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode != 0
    assert "WORLD_SIZE=1" in r.stderr

import json
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))

GOLDEN = ROOT / "tests" / "golden" / "ref_golden.json"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    return json.loads(GOLDEN.read_text())


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def cuda():
    """The CUDA path; on a GPU box a missing library is a hard failure (no fallback)."""
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test on a host without CUDA")
    from paper_1505_01120_b200 import capi

    capi.load()
    torch.cuda.set_device(0)
    return torch.device("cuda", 0)

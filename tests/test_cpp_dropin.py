"""The C++ drop-in (seam A GpuClusterDriver / seam B CudaExecutor) driven by
the UNMODIFIED reference Engine, compared bitwise with the reference host
executor (tests/cpp/test_dropin.cpp)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
EXE = ROOT / "build" / "test_dropin"


@pytest.mark.gpu
def test_cpp_dropin_parity():
    if not EXE.exists():
        pytest.fail(f"{EXE} missing: run __graft_entry__.build() where the reference headers exist")
    r = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:])
    print(r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "RESULT pass=" in r.stdout and "fail=0" in r.stdout


def test_cpp_dropin_built_or_reference_absent():
    """CPU: the drop-in compiled (it needs the reference headers, present here)."""
    if Path("/root/reference/proj/include/ucores/engine.hpp").exists():
        assert EXE.exists(), "build() must compile tests/cpp/test_dropin.cpp against the reference headers"

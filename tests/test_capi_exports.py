"""CPU: the C-ABI libraries load, export every symbol their headers declare,
the Python binding covers them, and with no GPU every compute entry fails
loudly (no CPU fallback)."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADERS = {"ucg_": ROOT / "include" / "ucores_cuda.h", "ucd_": ROOT / "include" / "ucores_engine.h"}
LIBS = {"ucg_": ROOT / "paper_1505_01120_b200" / "_lib" / "libucores_cuda.so",
        "ucd_": ROOT / "paper_1505_01120_b200" / "_lib" / "libucores_engine.so"}


def declared(prefix):
    text = HEADERS[prefix].read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(" + prefix + r"\w+)\s*\(", text)))


def exported(path):
    out = subprocess.run(["nm", "-D", "--defined-only", str(path)], capture_output=True, text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if line.strip()}


@pytest.mark.parametrize("prefix", ["ucg_", "ucd_"])
def test_library_exports_header(prefix):
    lib = LIBS[prefix]
    if not lib.exists():
        pytest.fail(f"{lib} not built: run __graft_entry__.build()")
    C.CDLL(str(lib))  # loads without a GPU
    missing = [s for s in declared(prefix) if s not in exported(lib)]
    assert not missing, missing
    assert len(declared(prefix)) >= (30 if prefix == "ucg_" else 3)


def test_python_binding_covers_header():
    from paper_1505_01120_b200 import capi

    assert set(declared("ucg_")) == set(capi.SIGNATURES), set(declared("ucg_")) ^ set(capi.SIGNATURES)


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1505_01120_b200 import DeviceUnavailable, capi

    lib = capi.load()
    assert capi.device_count() == 0
    assert lib.ucg_abi_version() == 1
    # compute entries refuse without a sm_100 device
    assert lib.ucg_map_affine_f32(None, None, 16, 2.0, 1.0, None) == capi.ERR_NODEV
    assert b"no CPU fallback" in lib.ucg_last_error()
    with pytest.raises(DeviceUnavailable):
        capi.call("ucg_tree_reduce_f32", None, 0, 0, None, None)
    from paper_1505_01120_b200 import ops

    x = torch.zeros(8)
    with pytest.raises(DeviceUnavailable):
        ops.map_affine(x, x, 2.0, 1.0)


def test_sm100a_code_only():
    """Every kernel in the library is sm_100a SASS (no PTX JIT / other arch)."""
    lib = LIBS["ucg_"]
    out = subprocess.run(["cuobjdump", "--list-elf", str(lib)], capture_output=True, text=True).stdout
    elfs = [l for l in out.splitlines() if "ELF file" in l]
    assert elfs and all("sm_100a" in l for l in elfs), out

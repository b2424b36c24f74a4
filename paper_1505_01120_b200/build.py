"""In-tree build of the native libraries (sm_100a only).

  _lib/libucores_cuda.so    CUDA kernels + runtime behind include/ucores_cuda.h
  _lib/libucores_engine.so  the C++ drop-in (seam A / seam B adapters and the
                            device-resident engine) compiled against the
                            UNMODIFIED reference headers; needs the reference
                            tree, so it is built here and travels prebuilt.

nvcc cross-compiles without a GPU. Built files are git-ignored but ship to the
GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
import sysconfig
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
HOST = PKG / "host"
LIB = PKG / "_lib"
OBJ = ROOT / "build" / "obj"
INCLUDE = ROOT / "include"
REF_INC = Path(os.environ.get("UCORES_REF_INC", "/root/reference/proj/include"))

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-I", str(INCLUDE),
                     "--expt-relaxed-constexpr"]

CUDA_SOURCES = ["ucg_runtime.cu", "ucg_reduce.cu", "ucg_pi.cu", "ucg_sobel.cu", "ucg_gemm.cu", "ucg_text.cu"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _site() -> Path:
    return Path(sysconfig.get_paths()["purelib"])


def json_include() -> Path:
    return _site() / "include" / "cudnn_frontend" / "thirdparty" / "nlohmann"


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps if d.exists())


def _run(cmd: list[str], verbose: bool) -> None:
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")


def build_cuda(force: bool = False, verbose: bool = False) -> Path:
    LIB.mkdir(parents=True, exist_ok=True)
    OBJ.mkdir(parents=True, exist_ok=True)
    nvcc = _nvcc()
    headers = list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))
    jobs = []
    objs = []
    for src in CUDA_SOURCES:
        s = CSRC / src
        o = OBJ / (s.stem + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append([nvcc] + NVCC_FLAGS + ["-c", str(s), "-o", str(o)])
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        list(ex.map(lambda c: _run(c, verbose), jobs))
    out = LIB / "libucores_cuda.so"
    if force or jobs or _stale(out, objs):
        _run([nvcc] + ARCH + ["-shared", "-o", str(out)] + [str(o) for o in objs], verbose)
    return out


def build_engine(force: bool = False, verbose: bool = False) -> Path | None:
    """The C++ drop-in; returns None when the reference headers are absent."""
    out = LIB / "libucores_engine.so"
    if not (REF_INC / "ucores" / "engine.hpp").exists():
        if not out.exists():
            print("reference headers absent: libucores_engine.so not built", file=sys.stderr)
        return out if out.exists() else None
    cuda_lib = build_cuda(force=False, verbose=verbose)
    srcs = [HOST / "engine_capi.cpp"]
    deps = srcs + list((HOST / "ucores_b200").glob("*.hpp")) + [cuda_lib] + list(INCLUDE.glob("*.h"))
    if not (force or _stale(out, deps)):
        return out
    cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-pthread", "-ffp-contract=off",
           "-I", str(REF_INC), "-I", str(json_include()), "-I", str(INCLUDE), "-I", str(HOST),
           "-I", "/usr/local/cuda/include",
           "-o", str(out)] + [str(s) for s in srcs] + [
           "-L", str(LIB), "-lucores_cuda", "-Wl,-rpath,$ORIGIN",
           "-L", "/usr/local/cuda/lib64", "-lcudart"]
    _run(cmd, verbose)
    return out


def build_tests(force: bool = False, verbose: bool = False) -> Path | None:
    """C++ drop-in test program (reference Engine + GPU seams)."""
    out = ROOT / "build" / "test_dropin"
    src = ROOT / "tests" / "cpp" / "test_dropin.cpp"
    if not src.exists() or not (REF_INC / "ucores" / "engine.hpp").exists():
        return out if out.exists() else None
    cuda_lib = build_cuda(force=False, verbose=verbose)
    deps = [src, cuda_lib] + list((HOST / "ucores_b200").glob("*.hpp")) + list(INCLUDE.glob("*.h"))
    if not (force or _stale(out, deps)):
        return out
    out.parent.mkdir(parents=True, exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-pthread", "-ffp-contract=off",
           "-I", str(REF_INC), "-I", str(json_include()), "-I", str(INCLUDE), "-I", str(HOST),
           "-I", "/usr/local/cuda/include",
           "-o", str(out), str(src),
           "-L", str(LIB), "-lucores_cuda", "-Wl,-rpath," + str(LIB),
           "-L", "/usr/local/cuda/lib64", "-lcudart"]
    _run(cmd, verbose)
    return out


def build_oracle(verbose: bool = False) -> None:
    """Test infrastructure: the C oracle and (when the reference tree exists) oracle/_ref."""
    _run(["make", "-s", "-C", str(ROOT / "oracle"), "all"], verbose)


def build_all(force: bool = False, verbose: bool = False) -> None:
    build_cuda(force, verbose)
    if (HOST / "engine_capi.cpp").exists():
        build_engine(force, verbose)
    build_tests(force, verbose)
    build_oracle(verbose)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv, verbose=True)

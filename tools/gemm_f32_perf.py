"""C5 GEMM rates at n = 8192 in one process: ucg_gemm_f32 (fp32-faithful
3xTF32, k-chunk sums in registers), ucg_gemm_tf32, cuBLAS TF32 and cuBLAS
SGEMM; CUDA events over 10 launches each after warm-up. One JSON line."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1505_01120_b200 import capi, ops  # noqa: E402


def rand(n, seed):
    t = torch.empty(n * n, dtype=torch.float32, device="cuda")
    ops.fill_uniform_(t, seed)
    return (t * 2 - 1).view(n, n)


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    capi.load()
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    A, B = rand(n, 100), rand(n, 101)
    Cm = torch.empty(n, n, device="cuda")
    fl = 2.0 * n ** 3
    out = {"n": n}
    out["f32_ms"] = timed(lambda: ops.gemm_f32(A, B, Cm, n))
    out["tf32_ms"] = timed(lambda: ops.gemm_tf32(A, B, Cm, n))
    torch.backends.cuda.matmul.allow_tf32 = True
    out["cublas_tf32_ms"] = timed(lambda: torch.matmul(A, B, out=Cm))
    torch.backends.cuda.matmul.allow_tf32 = False
    out["cublas_sgemm_ms"] = timed(lambda: torch.matmul(A, B, out=Cm), reps=3)
    for k in list(out):
        if k.endswith("_ms"):
            out[k.replace("_ms", "_tfs")] = fl / (out[k] * 1e-3) / 1e12
    out["f32_vs_cublas_tf32_over_3"] = out["f32_tfs"] / (out["cublas_tf32_tfs"] / 3)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

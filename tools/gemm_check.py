"""Dev check of ucg_gemm_tf32: accuracy vs fp64 and cuBLAS TF32, throughput at 8192."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1505_01120_b200 import capi, ops  # noqa: E402


def rand(n, seed):
    t = torch.empty(n * n, dtype=torch.float32, device="cuda")
    ops.fill_uniform_(t, seed)
    return (t * 2 - 1).view(n, n)


def main():
    res = {}
    for n in [256, 512, 1024, 2048]:
        A, B = rand(n, 100), rand(n, 101)
        Cm = torch.empty(n, n, dtype=torch.float32, device="cuda")
        ops.gemm_tf32(A, B, Cm, n)
        torch.cuda.synchronize()
        ref = (A.double() @ B.double())
        torch.backends.cuda.matmul.allow_tf32 = True
        cub = A @ B
        err = (Cm.double() - ref).abs()
        cerr = (cub.double() - ref).abs()
        res[n] = {"max_err": float(err.max()), "rms_err": float(err.pow(2).mean().sqrt()),
                  "cublas_tf32_max": float(cerr.max()), "cublas_tf32_rms": float(cerr.pow(2).mean().sqrt()),
                  "ref_rms": float(ref.pow(2).mean().sqrt())}
        print(n, res[n], flush=True)
    n = 8192
    A, B = rand(n, 100), rand(n, 101)
    Cm = torch.empty(n, n, dtype=torch.float32, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def t(fn, reps=10):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        return ts[len(ts) // 2]

    ms = t(lambda: ops.gemm_tf32(A, B, Cm, n))
    ms_f32 = t(lambda: ops.gemm_f32(A, B, Cm, n))
    torch.backends.cuda.matmul.allow_tf32 = True
    ms_cub = t(lambda: torch.matmul(A, B))
    torch.backends.cuda.matmul.allow_tf32 = False
    ms_fp32 = t(lambda: torch.matmul(A, B), reps=3)
    fl = 2 * n ** 3
    res["8192"] = {"ours_ms": ms, "ours_tflops": fl / ms / 1e9, "cublas_tf32_ms": ms_cub,
                   "cublas_tf32_tflops": fl / ms_cub / 1e9, "cublas_fp32_tflops": fl / ms_fp32 / 1e9,
                   "ours_3xtf32_ms": ms_f32, "ours_3xtf32_tflops": fl / ms_f32 / 1e9}
    idx = torch.randint(0, n, (64, 2), device="cuda")
    refv = torch.stack([(A[i].double() * B[:, j].double()).sum() for i, j in idx.tolist()])
    got = torch.stack([Cm[i, j].double() for i, j in idx.tolist()])
    res["8192"]["sampled_max_err_3xtf32"] = float((got - refv).abs().max())
    print(json.dumps(res["8192"]), flush=True)


if __name__ == "__main__":
    main()

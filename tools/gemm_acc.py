"""Accuracy of the GEMM modes vs an fp64 product (rms and max, relative to
rms(C64)): TF32, 3xTF32 (ucg_gemm_f32), cuBLAS SGEMM. Dev tool."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1505_01120_b200 import ops  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
for n in [int(v) for v in (sys.argv[1:] or ["256", "1024", "2048", "4096"])]:
    t = torch.empty(2 * n * n, dtype=torch.float32, device="cuda")
    ops.fill_uniform_(t, 100 + n)
    t = t * 2 - 1
    A, B = t[: n * n].view(n, n), t[n * n:].view(n, n)
    ref = A.double() @ B.double()
    rms = float(ref.pow(2).mean().sqrt())
    row = {}
    C = torch.empty(n, n, device="cuda")
    for name, fn in (("tf32", lambda: ops.gemm_tf32(A, B, C, n)), ("3xtf32", lambda: ops.gemm_f32(A, B, C, n)),
                     ("sgemm", lambda: C.copy_(A @ B))):
        fn()
        e = C.double() - ref
        row[name] = (float(e.pow(2).mean().sqrt()) / rms, float(e.abs().max()) / rms)
    print(n, " ".join(f"{k}: rms {v[0]:.2e} max {v[1]:.2e}" for k, v in row.items()), flush=True)

"""Dev: run one workload kernel a few times (for ncu captures)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1505_01120_b200 import ops  # noqa: E402

which = sys.argv[1]
if which == "sobel":
    H = W = 16384
    R = 256
    nb = H // R
    inp = torch.empty(nb * (R + 2) * W, dtype=torch.uint8, device="cuda")
    ops.fill_bytes_(inp, 7)
    out = torch.empty(H * W, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        ops.sobel_bands(inp, [b * (R + 2) * W for b in range(nb)], out, [b * R * W for b in range(nb)], [R] * nb, W)
elif which == "pi":
    hits = torch.empty(64, dtype=torch.int64, device="cuda")
    for _ in range(2):
        ops.pi_hits([42 + t for t in range(64)], [(1 << 30) // 64] * 64, hits)
elif which == "gemm_f32":
    n = 8192
    A = torch.randn(n, n, device="cuda")
    B = torch.randn(n, n, device="cuda")
    C = torch.empty(n, n, device="cuda")
    for _ in range(2):
        ops.gemm_f32(A, B, C, n)
elif which == "c1":
    from paper_1505_01120_b200.pipeline import MapReducePipeline

    pipe = MapReducePipeline([1 << 18] * 4, plant_max=False)
    for _ in range(4):
        pipe.step()
elif which == "gemm":
    n = 8192
    A = torch.randn(n, n, device="cuda")
    B = torch.randn(n, n, device="cuda")
    C = torch.empty(n, n, device="cuda")
    for _ in range(2):
        ops.gemm_tf32(A, B, C, n)
torch.cuda.synchronize()
print("ok", which)

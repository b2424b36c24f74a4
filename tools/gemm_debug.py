"""Dev: diagnose ucg_gemm_tf32 layouts on a small problem."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1505_01120_b200 import ops  # noqa: E402

n = 256
torch.manual_seed(0)
A = torch.randn(n, n, device="cuda")
B = torch.randn(n, n, device="cuda")
Cm = torch.full((n, n), 7.0, device="cuda")
ops.gemm_tf32(A, B, Cm, n)
torch.cuda.synchronize()
print("C stats: absmean", Cm.abs().mean().item(), "n7", (Cm == 7.0).sum().item(), "nz", (Cm == 0).sum().item())
print("C[0,:6]", Cm[0, :6].tolist())
cands = {"A@B": A @ B, "A@B.T": A @ B.T, "A.T@B": A.T @ B, "A.T@B.T": A.T @ B.T, "(A@B).T": (A @ B).T}
for k, v in cands.items():
    print(k, "rel err", ((Cm - v).norm() / v.norm()).item(), v[0, :4].tolist())
# single nonzero probes
for (i, kk, j) in [(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1), (5, 9, 37), (130, 200, 250)]:
    A = torch.zeros(n, n, device="cuda")
    B = torch.zeros(n, n, device="cuda")
    A[i, kk] = 1.0
    B[kk, j] = 1.0
    Cm.fill_(0)
    ops.gemm_tf32(A, B, Cm, n)
    torch.cuda.synchronize()
    nzs = (Cm != 0).nonzero().tolist()
    print(f"A[{i},{kk}]=1, B[{kk},{j}]=1 -> nonzeros at {nzs[:8]} (want [[{i},{j}]])")
    # B only: ones row
    A.zero_()
    A[i, :] = 1.0
    B.zero_()
    B[kk, j] = 1.0
    Cm.fill_(0)
    ops.gemm_tf32(A, B, Cm, n)
    torch.cuda.synchronize()
    print(f"   A row {i} ones, B[{kk},{j}]=1 -> nonzeros {(Cm != 0).nonzero().tolist()[:8]}")

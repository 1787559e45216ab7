"""Where does the tcgen05 GEMM error come from? bf16-exact A (one plane) vs the
3-plane split; errors vs fp64."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_08723_b200 import kernels as K
torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda")
m, n, k = 480, 5000, 2048
torch.manual_seed(0)
a = torch.randn(m, k, device=dev) * 0.5
w = (torch.rand(n, k, device=dev) * 0.7 - 0.35).to(torch.bfloat16).float()
ab = a.to(torch.bfloat16).float()
for name, A, planes in (("bf16 A, 1 plane", ab, 1), ("bf16 A, 3 planes", ab, 3),
                        ("fp32 A, 3 planes", a, 3)):
    ap = torch.empty((3, m, k), dtype=torch.bfloat16, device=dev)
    K.pack(ap, [(A, k, 0)], m=m, k_pad=k, split=True)
    out = torch.zeros(m, n, device=dev)
    g = ap[:planes]
    K.gemm_tc(g.contiguous(), w.to(torch.bfloat16), m=m, k=k, out=out)
    ref = A.double() @ w.double().T
    e = out.double() - ref
    f = (A @ w.T).double() - ref
    print(f"{name:18s} tc std {e.std().item():.2e} max {e.abs().max().item():.2e} | "
          f"fp32 std {f.std().item():.2e}")
# k-dependence, bf16 exact single plane
for k2 in (64, 256, 1024, 4096):
    a2 = (torch.randn(m, k2, device=dev) * 0.5).to(torch.bfloat16).float()
    w2 = (torch.rand(1024, k2, device=dev) * 0.7 - 0.35).to(torch.bfloat16).float()
    ap = torch.empty((1, m, k2), dtype=torch.bfloat16, device=dev)
    ap[0] = a2.to(torch.bfloat16)
    out = torch.zeros(m, 1024, device=dev)
    K.gemm_tc(ap, w2.to(torch.bfloat16), m=m, k=k2, out=out)
    ref = a2.double() @ w2.double().T
    e = out.double() - ref
    f = (a2 @ w2.T).double() - ref
    print(f"k={k2:5d} tc std {e.std().item():.2e} fp32 std {f.std().item():.2e} ratio {e.std().item() / f.std().item():.1f}")

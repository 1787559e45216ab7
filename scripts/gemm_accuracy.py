"""Accuracy of the tcgen05 bf16x3 GEMM vs fp64 and vs torch fp32 (CUDA cores,
TF32 off) on decoder-shaped problems: error std / max / mean (bias)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_08723_b200 import kernels as K
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import testkit as TK
torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda")
for (m, n, k, sa, sw) in [(480, 5000, 2048, 0.5, 0.35), (480, 4096, 2304, 0.5, 1 / 32),
                          (480, 5000, 832, 0.5, 0.5)]:
    torch.manual_seed(0)
    a = torch.randn(m, k, device=dev) * sa
    w = (torch.rand(n, k, device=dev) * 2 * sw - sw).to(torch.bfloat16).float()
    ap = torch.empty((3, m, k), dtype=torch.bfloat16, device=dev)
    K.pack(ap, [(a, k, 0)], m=m, k_pad=k, split=True)
    out = torch.zeros(m, n, device=dev)
    K.gemm_tc(ap, w.to(torch.bfloat16), m=m, k=k, out=out)
    ref = a.double() @ w.double().T
    f32 = (a @ w.T).double()
    simt = torch.zeros(m, n, device=dev)
    TK.gemm(a, w, m=m, k=k, out=simt)
    for name, x in (("tc", out.double()), ("torch32", f32), ("simt", simt.double())):
        e = x - ref
        print(f"m{m} n{n} k{k}: {name:8s} std {e.std().item():.2e} max {e.abs().max().item():.2e} "
              f"mean {e.mean().item():+.2e}  (|ref| std {ref.std().item():.2f})")
    # planes: how exact is the split?
    rec = ap[0].double() + ap[1].double() + ap[2].double()
    print("   split residual max", (rec - a.double()).abs().max().item())

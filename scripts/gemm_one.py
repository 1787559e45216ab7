"""One tcgen05 GEMM shape, repeated (for ncu source-level captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_08723_b200 import kernels as K
M, N, Kd, P = (int(x) for x in os.environ.get("SHAPE", "5120,1280,1024,1").split(","))
dev = torch.device("cuda")
a = torch.randn(P, M, Kd, device=dev).to(torch.bfloat16)
w = (torch.randn(N, Kd, device=dev) * 0.05).to(torch.bfloat16)
out = torch.empty(M, N, device=dev)
for _ in range(5):
    K.gemm_tc(a, w, m=M, k=Kd, out=out, kcb=4)
torch.cuda.synchronize()

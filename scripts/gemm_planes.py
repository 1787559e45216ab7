"""Is the tcgen05 GEMM bound by its operand fill?  Time the same shape with
1, 2 and 3 A planes (A bytes per K block 16/32/48 KB; MMA work 1x/2x/3x)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_08723_b200 import kernels as K
dev = torch.device("cuda")
for (M, N, Kd) in ((5120, 1280, 1024), (2048, 1280, 1024), (160, 4800, 2432), (256, 65003, 1216)):
    a = torch.randn(3, M, Kd, device=dev).to(torch.bfloat16)
    w = (torch.randn(N, Kd, device=dev) * 0.05).to(torch.bfloat16)
    out = torch.empty(M, N, device=dev)
    for planes in (1, 2, 3):
        ap = a[:planes].contiguous()
        for _ in range(3):
            K.gemm_tc(ap, w, m=M, k=Kd, out=out, kcb=4)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()          # eager ctypes launches are host-bound
        with torch.cuda.graph(graph):
            for _ in range(20):
                K.gemm_tc(ap, w, m=M, k=Kd, out=out, kcb=4)
        graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        graph.replay()
        e1.record()
        torch.cuda.synchronize()
        us = 1000 * e0.elapsed_time(e1) / 20
        print(f"M{M} N{N} K{Kd} planes {planes}: {us:.1f} us  ({2 * M * N * Kd * planes / us / 1e6:.0f} TFLOP/s tensor)")

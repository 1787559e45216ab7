"""Where does the tcgen05 GEMM time go?  Vary planes / epilogue / K."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_08723_b200 import kernels as K

def t(M, N, Kd, planes, mode, reps=20):
    dev = torch.device("cuda")
    a = torch.randn(planes, M, Kd, device=dev).to(torch.bfloat16)
    w = (torch.randn(N, Kd, device=dev) * 0.05).to(torch.bfloat16)
    if mode == 1:
        H = N // 4
        kw = dict(mode=1, hidden=H, c_in=torch.randn(M, H, device=dev),
                  c_out=torch.empty(M, H, device=dev), h_out=torch.empty(M, H, device=dev))
    else:
        kw = dict(out=torch.empty(M, N, device=dev))
    K.gemm_tc(a, w, m=M, k=Kd, **kw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        K.gemm_tc(a, w, m=M, k=Kd, **kw)
    e1.record(); torch.cuda.synchronize()
    us = 1000 * e0.elapsed_time(e1) / reps
    return us, 2.0 * M * N * Kd * planes / (us * 1e-6) / 1e12

for (M, N, Kd) in [(5120, 1280, 1024), (5120, 1280, 4096), (16384, 1280, 1024)]:
    for planes in (1, 3):
        for mode in (0, 1):
            us, tf = t(M, N, Kd, planes, mode)
            print(f"M={M} N={N} K={Kd} planes={planes} mode={mode}: {us:8.1f} us  tensor {tf:7.1f} TF/s", flush=True)

"""Epilogue cost of the tcgen05 GEMM: same shape, plain stores (mode 0) vs the
LSTM-cell epilogue (mode 1, with/without row/parent gathers)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_08723_b200 import kernels as K
dev = torch.device("cuda")


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return 1000 * e0.elapsed_time(e1) / reps


for (M, N, Kd) in ((5120, 1280, 1024), (256, 4800, 2432)):
    H = N // 4
    ap = torch.randn(3, M, Kd, device=dev).to(torch.bfloat16)
    w = (torch.randn(N, Kd, device=dev) * 0.05).to(torch.bfloat16)
    b = torch.randn(N, device=dev)
    out = torch.empty(M, N, device=dev)
    c_in, c_out, h_out = (torch.randn(M, H, device=dev) for _ in range(3))
    rows = torch.randperm(M, device=dev).to(torch.int32)
    par = torch.randperm(M, device=dev).to(torch.int32)
    for kcb in (4, 16):
        r = {
            "mode0": t(lambda: K.gemm_tc(ap, w, m=M, k=Kd, out=out, kcb=kcb)),
            "mode0_bias": t(lambda: K.gemm_tc(ap, w, m=M, k=Kd, bias=b, out=out, kcb=kcb)),
            "lstm": t(lambda: K.gemm_tc(ap, w, m=M, k=Kd, bias=b, mode=1, hidden=H, c_in=c_in,
                                        c_out=c_out, h_out=h_out, kcb=kcb)),
            "lstm_gather": t(lambda: K.gemm_tc(ap, w, m=M, k=Kd, bias=b, mode=1, hidden=H,
                                               c_in=c_in, c_out=c_out, h_out=h_out, rows=rows,
                                               parent=par, kcb=kcb)),
        }
        print(f"M{M} N{N} K{Kd} kcb {kcb}: " + "  ".join(f"{k} {v:.1f}us" for k, v in r.items()))

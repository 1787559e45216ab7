"""Per-k-block event times of CTA 0 in one tcgen05 GEMM (library built with
FB_NVCC_EXTRA=-DFB_GEMM_TRACE): producer wait on 'empty', MMA wait on 'full'."""
import ctypes as C
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1909_08723_b200 import _lib, kernels as K
M, N, Kd, P = (int(x) for x in os.environ.get("SHAPE", "5120,1280,1024,3").split(","))
dev = torch.device("cuda")
a = torch.randn(P, M, Kd, device=dev).to(torch.bfloat16)
w = (torch.randn(N, Kd, device=dev) * 0.05).to(torch.bfloat16)
out = torch.empty(M, N, device=dev)
sk = K.SplitK(dev) if os.environ.get("SPLITK") == "1" else None
for _ in range(3):
    K.gemm_tc(a, w, m=M, k=Kd, out=out, kcb=4, splitk=sk)
torch.cuda.synchronize()
buf = np.zeros((10, 256), np.uint64)
lib = C.CDLL(_lib.LIB_PATH)
lib.fb_gemm_trace_read(buf.ctypes.data)
t0 = buf[0, 0]
tr = (buf.astype(np.int64) - int(t0)) / 1000.0      # us
nk = min(48, int((buf[4] > 0).sum()))
print("kb  prod_wait_start  prod_issue  mma_wait_start  mma_full  mma_commit   (us from first)")
for i in range(nk):
    print(f"{i:3d} {tr[0, i]:8.2f} {tr[1, i]:8.2f} {tr[2, i]:8.2f} {tr[3, i]:8.2f} {tr[4, i]:8.2f}")
print("segment  acc_ready  fixup_done  epilogue_done")
for i in range(8):
    if buf[7, i] > 0:
        print(f"{i:3d} {tr[5, i]:8.2f} {tr[6, i]:8.2f} {tr[7, i]:8.2f}")
print("epilogue chunk marks", [round(float(x), 2) for x in tr[8, :16]])

"""Per-k-block event times of CTA 0 in one tcgen05 GEMM (library built with
FB_BUILD_TAG=trace FB_NVCC_EXTRA=-DFB_GEMM_TRACE, loaded with FB_LIB_AB):
producer wait on 'empty' / issue, MMA wait on 'full' / commit, and the
epilogue's drain of each accumulation chunk.  SHAPE=M,N,K  MODE=0|1  KCB=n"""
import ctypes as C
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1909_08723_b200 import _lib, kernels as K  # noqa: E402

M, N, Kd = (int(x) for x in os.environ.get("SHAPE", "5120,1280,1024").split(","))
mode = int(os.environ.get("MODE", "1"))
kcb = int(os.environ.get("KCB", "1"))
dev = torch.device("cuda")
a = K.operand_planes(M, Kd, dev)
K.pack(a, [(torch.randn(M, Kd, device=dev), Kd, 0)], m=M, k_pad=Kd, split=True)
w = K.operand_weight(torch.randn(N, Kd, device=dev) * 0.05)
b = torch.randn(N, device=dev)
if mode == 1:
    H = N // 4
    kw = dict(mode=1, hidden=H, c_in=torch.randn(M, H, device=dev),
              c_out=torch.empty(M, H, device=dev), h_out=torch.empty(M, H, device=dev))
elif mode == 2:                  # logits + softmax tile statistics (the word-LM output)
    kw = dict(out=torch.empty(M, (N + 3) // 4 * 4, device=dev)[:, :N],
              row_stats=torch.empty(M, (N + 63) // 64, 4, device=dev), stats_vw=N - 3)
else:
    kw = dict(out=torch.empty(M, (N + 3) // 4 * 4, device=dev)[:, :N])
for _ in range(3):
    K.gemm_tc(a, w, m=M, k=Kd, bias=b, kcb=kcb, **kw)
torch.cuda.synchronize()
buf = np.zeros((10, 256), np.uint64)
lib = C.CDLL(_lib.LIB_PATH)
lib.fb_gemm_trace_read(buf.ctypes.data)
t0 = buf[0, 0]
tr = (buf.astype(np.int64) - int(t0)) / 1000.0      # us
nk = min(40, int((buf[4] > 0).sum()))
print("kb  prod_wait_start  prod_issue  mma_wait_start  mma_full  mma_commit  chunk_drained (us)")
for i in range(nk):
    print(f"{i:3d} {tr[0, i]:8.2f} {tr[1, i]:8.2f} {tr[2, i]:8.2f} {tr[3, i]:8.2f} {tr[4, i]:8.2f}"
          f" {tr[9, i]:8.2f}")
print("segment  acc_ready  fixup_done  epilogue_done")
for i in range(int(os.environ.get("SEGS", "4"))):
    if buf[7, i] > 0:
        print(f"{i:3d} {tr[5, i]:8.2f} {tr[6, i]:8.2f} {tr[7, i]:8.2f}")
print("epilogue chunk marks (start/end per 32-column chunk, last warp to write)",
      [round(float(x), 2) for x in tr[8, :8]])

"""Per-step phases of CTA 0 in the persistent encoder recurrence (build with
FB_NVCC_EXTRA=-DFB_GEMM_TRACE): barrier wait, mainloop, epilogue."""
import ctypes as C
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1909_08723_b200 import _lib
B, H, TM = 512, 320, 225
k = 320
dev = torch.device("cuda")
w = (torch.randn(4 * H, k, device=dev) * 0.05).to(torch.bfloat16)
xp = torch.randn(B, TM, 4 * H, device=dev) * 0.1
y = torch.empty(B, TM, H, device=dev)
cb = torch.empty(2, B, H, device=dev)
rec = torch.zeros(2, 3, B, k, dtype=torch.bfloat16, device=dev)
sync = torch.zeros(1, dtype=torch.int32, device=dev)
TMAJOR = os.environ.get("TMAJOR") == "1"     # time-major xp / y (rows of a step contiguous)
for _ in range(2):
    rec.zero_()
    if os.environ.get("XPZERO") == "1":        # every row reads the same xp row (cache hits)
        _lib.call("fb_lstm_recurrence", TM, B, H, _lib.ptr(w), k, _lib.ptr(xp), 0,
                  0, _lib.ptr(y), TM * H, H, _lib.ptr(rec), _lib.ptr(sync),
                  _lib.stream_ptr())
    elif TMAJOR:
        _lib.call("fb_lstm_recurrence", TM, B, H, _lib.ptr(w), k, _lib.ptr(xp), 4 * H,
                  B * 4 * H, _lib.ptr(y), H, B * H, _lib.ptr(rec), _lib.ptr(sync),
                  _lib.stream_ptr())
    else:
        _lib.call("fb_lstm_recurrence", TM, B, H, _lib.ptr(w), k, _lib.ptr(xp), TM * 4 * H,
                  4 * H, _lib.ptr(y), TM * H, H, _lib.ptr(rec), _lib.ptr(sync),
                  _lib.stream_ptr())
torch.cuda.synchronize()
buf = np.zeros((10, 256), np.uint64)
C.CDLL(_lib.LIB_PATH).fb_gemm_trace_read(buf.ctypes.data)
tr = (buf.astype(np.int64) - int(buf[0, 0])) / 1000.0
print("t   barrier_wait_start  barrier_pass  epi_start  epi_done  fenced  published   (us)")
for t in list(range(0, 6)) + list(range(100, 106)):
    print(f"{t:3d} {tr[0, t]:9.2f} {tr[1, t]:9.2f} {tr[2, t]:9.2f} {tr[4, t]:9.2f} {tr[5, t]:9.2f} {tr[3, t]:9.2f}")
print("mean step", (tr[3, 200] - tr[3, 100]) / 100)

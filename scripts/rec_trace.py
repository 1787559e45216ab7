"""Encoder recurrence timing at the c2 shape (B=512, T=225, H=320, k=320):
one direction alone, both directions on two streams (as the encoder runs
them), and -- with a trace build (FB_BUILD_TAG=trace FB_NVCC_EXTRA=-DFB_GEMM_TRACE,
FB_LIB_AB=libfusedbeam_b200_trace.so) -- the per-step phases of CTA 0:
barrier wait, barrier pass, accumulator drained, stores done, fenced, published.
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1909_08723_b200 import _lib, kernels as K  # noqa: E402

B, H, TM = int(os.environ.get("B", 512)), 320, 225
k = 320
dev = torch.device("cuda")
planes = K.operand_format()[0]
w = [K.operand_weight(torch.randn(4 * H, k, device=dev) * 0.05) for _ in range(2)]
xp = torch.randn(B, TM, 8 * H, device=dev) * 0.1
y = torch.empty(B, TM, 2 * H, device=dev)
rec = [torch.zeros(2, planes, B, k, dtype=K.operand_format()[1], device=dev) for _ in range(2)]
sync = [torch.zeros(32 * 8, dtype=torch.int32, device=dev) for _ in range(2)]
t_rev = torch.full((B,), TM, dtype=torch.int32, device=dev)
streams = [torch.cuda.Stream(), torch.cuda.Stream()]


def launch(r, stream):
    rec[r].zero_()
    _lib.call("fb_lstm_recurrence", TM, B, H, _lib.ptr(w[r]), k,
              _lib.ptr(xp) + 4 * (4 * H) * r, TM * 8 * H, 8 * H,
              _lib.ptr(y) + 4 * H * r, TM * 2 * H, 2 * H, _lib.ptr(rec[r]), _lib.ptr(sync[r]),
              w[r].fb_acc_scale, _lib.ptr(t_rev) if r == 1 else None, int(stream.cuda_stream))


def timed(dirs):
    main = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        e0.record(main)
        for r in dirs:
            streams[r].wait_stream(main)
            with torch.cuda.stream(streams[r]):
                launch(r, streams[r])
        for r in dirs:
            main.wait_stream(streams[r])
        e1.record(main)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1000)
    return best


one = timed([0])
both = timed([0, 1])
print(f"B={B}: one direction {one:.0f} us ({one / TM:.2f} us/step); both directions on two "
      f"streams {both:.0f} us ({both / TM:.2f} us/step)")
lib = C.CDLL(_lib.LIB_PATH)
if hasattr(lib, "fb_gemm_trace_read"):
    timed([0])
    buf = np.zeros((10, 256), np.uint64)
    lib.fb_gemm_trace_read(buf.ctypes.data)
    tr = (buf.astype(np.int64) - int(buf[0, 0])) / 1000.0
    print("t   wait_start  barrier_pass  acc_drained  stored  fenced  published   (us)")
    for t in list(range(0, 4)) + list(range(100, 104)):
        print(f"{t:3d} {tr[0, t]:9.2f} {tr[1, t]:9.2f} {tr[2, t]:9.2f} {tr[4, t]:9.2f} "
              f"{tr[5, t]:9.2f} {tr[3, t]:9.2f}")
    s = slice(50, 200)
    print("mean over t=50..199: pass-after-publish(t-1) %.2f, drained-after-pass %.2f, "
          "stored %.2f, fenced %.2f, published %.2f, step %.2f us" % (
              np.mean(tr[1, 50:200] - tr[3, 49:199]), np.mean(tr[2, s] - tr[1, s]),
              np.mean(tr[4, s] - tr[2, s]), np.mean(tr[5, s] - tr[4, s]),
              np.mean(tr[3, s] - tr[5, s]), (tr[3, 199] - tr[3, 49]) / 150))
    # per-CTA: publish of step 100, barrier wait start / pass of step 101 (CTA = m-tile + 4 n)
    n = (B + 127) // 128 * 10
    pub, ws, ps = tr[9, :n], tr[6, :n], tr[7, :n]
    m_tiles = (B + 127) // 128
    for m in range(m_tiles):
        idx = list(range(m, n, m_tiles))
        print(f"m-tile {m}: publish(100) spread {pub[idx].max() - pub[idx].min():.2f} us "
              f"(first {pub[idx].min():.2f}, last {pub[idx].max():.2f}); pass(101) "
              f"{ps[idx].min():.2f}..{ps[idx].max():.2f}; last publish -> first pass "
              f"{ps[idx].min() - pub[idx].max():.2f} us")
    sm = buf[8, :n].astype(np.int64)
    print("per CTA (m-tile 0..3 interleaved): cta sm wait_start(101) publish(100) pass(101)")
    for i in np.argsort(ps)[:: max(1, n // 20)]:
        print(f"  {i:3d} sm{sm[i]:3d} {ws[i]:9.2f} {pub[i]:9.2f} {ps[i]:9.2f}")
    late = ps - ps.min()
    print("pass(101) lateness vs sm id: corr", np.corrcoef(sm, late)[0, 1])

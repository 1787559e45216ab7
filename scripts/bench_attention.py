"""Time fb_attention_step (query exp + energy + context/accumulator) alone at
the c2 and c4 decoder shapes (all rows live, longest T), CUDA events."""
import ctypes as C
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_08723_b200 import _lib

if os.environ.get("FB_LIB"):                 # A/B against another build of the library
    _lib.LIB_PATH = os.environ["FB_LIB"]
    _h = C.CDLL(_lib.LIB_PATH)
    for _name in list(_lib._SIGS):
        if not hasattr(_h, _name):
            del _lib._SIGS[_name]
P = _lib.ptr
dev = torch.device("cuda")
for name, B, K, T, A, Cd in (("c2", 512, 10, 225, 320, 640), ("c4", 32, 60, 875, 512, 1024)):
    torch.manual_seed(0)
    N = B * K
    cfg = _lib.FbSearchCfg(beam=K, vocab=52, t_max=T, cov_mode=0)
    active = torch.ones(B, dtype=torch.int32, device=dev)
    n_live = torch.full((B,), K, dtype=torch.int32, device=dev)
    t_enc = torch.full((B,), T, dtype=torch.int32, device=dev)
    keys = torch.exp(2 * torch.randn(B * T, A, device=dev) * 0.5)
    enc = torch.randn(B * T, Cd, device=dev)
    v = torch.randn(A, device=dev) * 0.1
    q0 = torch.randn(N, A, device=dev) * 0.5
    q = q0.clone()
    parent = torch.arange(N, dtype=torch.int32, device=dev)
    acc_in = torch.zeros(N, T, dtype=torch.float64, device=dev)
    acc_out = torch.zeros_like(acc_in)
    ctx = torch.zeros(N, Cd, device=dev)
    energy = torch.zeros(2, N, T, device=dev)
    sync = torch.zeros(B * ((K + 1) // 2), dtype=torch.int32, device=dev)

    def run():
        q.copy_(q0)
        _lib.call("fb_attention_step", C.byref(cfg), B, P(active), P(n_live), P(t_enc), P(keys),
                  P(enc), A, Cd, P(v), P(q), A, P(parent), P(acc_in), P(acc_out), None, P(ctx),
                  Cd, None, 0, P(energy), P(sync), 0, None, 0, 0, None, _lib.stream_ptr())
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    R = 20
    for _ in range(R):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / R
    elems = N * T * A
    print(f"{name}: {ms * 1000:.1f} us per attention step; energy elems {elems / 1e6:.0f}M "
          f"(MUFU floor 1 rcp/elem {elems / (16 * 148 * 1.9e9) * 1e6:.0f} us), enc bytes "
          f"{B * T * Cd * 4 / 1e6:.0f} MB (HBM floor {B * T * Cd * 4 / 7.0e12 * 1e6:.0f} us)")

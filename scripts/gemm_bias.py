"""Signed error of the tensor-core projections against fp64, on the c5 and c2
acoustic output shapes (weights and activation ranges of the real models):
is the accumulated per-step score drift of long decodes a bias of the logits
(TMEM accumulation) or of the log-softmax?

    python scripts/gemm_bias.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import harness as H  # noqa: E402
from paper_1909_08723_b200 import kernels as K  # noqa: E402
from paper_1909_08723_b200.models import _devw  # noqa: E402

dev = torch.device("cuda")
for name in ("c2", "c5", "c4"):
    wl = H.workload(name)
    S = H.synth()
    W = S.asr_weights(wl.asr, seed=wl.seed, eos_id=1)
    w = torch.as_tensor(W["dec.out.w"], device=dev)          # [V, H + C]
    b = torch.as_tensor(W["dec.out.b"], device=dev)
    V, Kd = w.shape
    kp = (Kd + 63) // 64 * 64
    m = 4096
    torch.manual_seed(0)
    # h: LSTM outputs (+ residuals, |h| < 3), ctx: attention over BiLSTM outputs (|ctx| < 1)
    Hd = wl.asr.dec_hidden
    x = torch.cat([torch.tanh(torch.randn(m, Hd, device=dev)) * 1.5,
                   torch.tanh(torch.randn(m, Kd - Hd, device=dev) * 0.5)], dim=1)
    ap = K.operand_planes(m, kp, dev)
    K.pack(ap, [(x, Kd, 0)], m=m, k_pad=kp, split=True)
    wp = _devw(W["dec.out.w"], dev, kp)
    out = torch.empty(m, V, device=dev)
    K.gemm_tc(ap, wp, m=m, k=kp, bias=b, out=out, kcb=1)
    ref = x.double() @ w.double().T + b.double()
    err = out.double() - ref
    am = ref.argmax(dim=1)
    e_top = err.gather(1, am[:, None])[:, 0]
    lp_ref = torch.log_softmax(ref, dim=1)
    lp_gpu = torch.empty(m, V, device=dev)
    K.log_softmax_rows(out, lp_gpu, V, m=m)
    lerr = (lp_gpu.double() - lp_ref).gather(1, am[:, None])[:, 0]
    lp32 = torch.log_softmax(out, dim=1).double()                # torch fp32 log-softmax
    lerr32 = (lp32 - lp_ref).gather(1, am[:, None])[:, 0]
    # torch fp32 CPU logits (the oracle's arithmetic) for comparison
    cpu = (x.cpu() @ w.cpu().T + b.cpu()).double()
    cerr = (cpu - ref.cpu()).gather(1, am.cpu()[:, None])[:, 0]
    print(f"{name}: V={V} K={Kd} |logit|max {ref.abs().max().item():.1f}; GEMM err: mean "
          f"{err.mean().item():+.3g} top-logit mean {e_top.mean().item():+.3g} max|.| "
          f"{err.abs().max().item():.3g}; logp(top) err mean {lerr.mean().item():+.3g} "
          f"(torch-fp32 lsm on GPU logits {lerr32.mean().item():+.3g}); CPU fp32 top-logit err "
          f"mean {cerr.mean().item():+.3g} max {cerr.abs().max().item():.3g}")

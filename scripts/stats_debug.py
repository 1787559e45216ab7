"""Debug the LM-output tile statistics on a multi-m-tile shape."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_1909_08723_b200 import kernels as K
import test_gpu_gemm as T
dev = torch.device("cuda")
for m, vw, k in [(37, 9000, 128), (300, 9000, 128), (300, 65000, 1216), (130, 65000, 128)]:
    torch.manual_seed(11 + m)
    n = vw + 3
    a = torch.randn(m, k, device=dev)
    w = T._bf16_exact(torch.randn(n, k, device=dev) * 0.3)
    b = torch.randn(n, device=dev) * 0.5
    logits = torch.empty(m, n, device=dev)
    stats = torch.full((m, (n + 63) // 64, 4), float("nan"), device=dev)
    K.gemm_tc(T._packed(a, k), T._w(w), m=m, k=k, bias=b, out=logits, row_stats=stats, stats_vw=vw)
    torch.cuda.synchronize()
    nt = (n + 63) // 64
    L = torch.nn.functional.pad(logits, (0, nt * 64 - n), value=float("-inf")).view(m, nt, 64)
    mx = L.max(dim=2).values
    se = torch.exp(L - mx[..., None]).sum(dim=2)
    bad_nan = torch.isnan(stats[..., 0]).sum().item()
    dm = (stats[..., 0] - mx).abs().nan_to_num(1e9)
    ds = ((stats[..., 1] - se) / se).abs().nan_to_num(1e9)
    rows_bad = ((dm > 1e-4) | (ds > 1e-4)).any(dim=1).nonzero().flatten().tolist()
    print(m, vw, k, "nan tiles", bad_nan, "bad rows", len(rows_bad), rows_bad[:10],
          "max dm", dm.max().item(), "max ds", ds.max().item(), flush=True)

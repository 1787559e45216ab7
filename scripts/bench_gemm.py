"""Standalone timing of the tcgen05 GEMM at the decoder's shapes (CUDA events,
graph-captured, rotating 4 operand sets).  Algorithmic FLOPs = 2*M*N*K (the
operand planes are not counted).  KCB=n: TMEM accumulation chunk."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_08723_b200 import kernels as K

SHAPES = {  # name: (M, N, K, mode)
    "lm_lstm_64": (64, 4800, 2432, 1),
    "lm_lstm_300": (300, 4800, 2432, 1),
    "am_lstm_2k": (2048, 1280, 1024, 1),
    "lm_lstm_160": (160, 4800, 2432, 1),
    "lm_lstm_600": (600, 4800, 2432, 1),
    "am_lstm": (5120, 1280, 1024, 1),
    "lm_lstm": (256, 4800, 2432, 1),
    "lm_out": (256, 65003, 1216, 0),
    "lm_out_240": (240, 65003, 1216, 2),      # mode 2: logits + softmax tile statistics
    "enc_proj": (115200, 1280, 320, 0),
    "enc_rec": (512, 1280, 320, 1),
    "am_q": (5120, 320, 320, 0),
    "am_out": (5120, 52, 640, 0),
    "am_out_2k": (2048, 52, 640, 0),
}

def run(name, M, N, Kd, mode, reps=20):
    dev = torch.device("cuda")
    sets = []
    nsets = int(os.environ.get("SETS", "4"))
    for _ in range(nsets):
        a = K.operand_planes(M, Kd, dev)
        K.pack(a, [(torch.randn(M, Kd, device=dev), Kd, 0)], m=M, k_pad=Kd, split=True)
        w = K.operand_weight(torch.randn(N, Kd, device=dev) * 0.05)
        b = torch.randn(N, device=dev)
        if mode == 1:
            H = N // 4
            kw = dict(mode=1, hidden=H, c_in=torch.randn(M, H, device=dev),
                      c_out=torch.empty(M, H, device=dev), h_out=torch.empty(M, H, device=dev))
        elif mode == 2:
            # rows padded to 16 bytes like the engine's event logits (TMA stores)
            kw = dict(out=torch.empty(M, (N + 3) // 4 * 4, device=dev)[:, :N],
                      row_stats=torch.empty(M, (N + 63) // 64, 4, device=dev), stats_vw=N - 3)
        else:
            kw = dict(out=torch.empty(M, (N + 3) // 4 * 4, device=dev)[:, :N])
        kw["kcb"] = int(os.environ.get("KCB", "0"))
        sets.append((a, w, b, kw))
    if os.environ.get("FB_BENCH_SPLITK") == "1":
        sk = K.SplitK(dev)
        for _, _, _, kw in sets:
            kw["splitk"] = sk
    for a, w, b, kw in sets:
        K.gemm_tc(a, w, m=M, k=Kd, bias=b, **kw)
    torch.cuda.synchronize()
    # captured in a CUDA graph: eager launches through ctypes are host-bound
    # (~35 us each), far above the small shapes' device time
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for i in range(reps):
            a, w, b, kw = sets[i % nsets]
            K.gemm_tc(a, w, m=M, k=Kd, bias=b, **kw)
    graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    graph.replay()
    e1.record()
    torch.cuda.synchronize()
    us = 1000 * e0.elapsed_time(e1) / reps
    tf = 2.0 * M * N * Kd / (us * 1e-6) / 1e12
    return {"shape": name, "M": M, "N": N, "K": Kd, "us": round(us, 2),
            "alg_tflops": round(tf, 1),
            "tensor_tflops_planes": round(K.operand_format()[0] * tf, 1)}

if __name__ == "__main__":
    names = sys.argv[1:] or list(SHAPES)
    for n in names:
        print(json.dumps(run(n, *SHAPES[n])), flush=True)

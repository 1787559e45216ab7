"""tcgen05 GEMM (split fp32 activations in the library's operand format --
two fp16 planes by default --, exact weights, fp32 TMEM accumulate) vs a plain
PyTorch fp64 reference of the same op; epilogues vs the fp32 SIMT kernel."""

import numpy as np
import pytest

import testkit as TK

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu(cuda_lib):
    return cuda_lib


def _bf16_exact(t):
    return t.to(torch.bfloat16).to(torch.float32)


def _packed(a, k_pad):
    from paper_1909_08723_b200 import kernels as K
    m = a.shape[0]
    out = K.operand_planes(m, k_pad, a.device)
    K.pack(out, [(a, a.shape[1], 0)], m=m, k_pad=k_pad, split=True)
    return out


def _w(w):
    from paper_1909_08723_b200 import kernels as K
    return K.operand_weight(w)


def _split_ref(h):
    """The operand planes of fp32 values h (common.cuh split_operand)."""
    from paper_1909_08723_b200 import kernels as K
    planes, dt, act = K.operand_format()
    y = h * act
    if planes == 2:
        hi = y.to(torch.float16)
        return [hi, (y - hi.float()).to(torch.float16)]
    hi = y.to(torch.bfloat16)
    r1 = y - hi.float()
    mid = r1.to(torch.bfloat16)
    return [hi, mid, (r1 - mid.float()).to(torch.bfloat16)]


@pytest.mark.parametrize("m,n,k", [(1, 52, 64), (70, 128, 1024), (128, 320, 320),
                                   (300, 1280, 1024), (129, 4800, 2432), (200, 65003, 1216)])
def test_tc_gemm_matches_fp64_reference(m, n, k):
    from paper_1909_08723_b200 import kernels as K
    torch.manual_seed(m + n + k)
    dev = torch.device("cuda")
    a = torch.randn(m, k, device=dev) * 0.5
    w = _bf16_exact(torch.rand(n, k, device=dev) * 0.2 - 0.1)
    b = torch.randn(n, device=dev)
    ap = _packed(a, k)
    out = torch.zeros(m, n, device=dev)
    K.gemm_tc(ap, _w(w), m=m, k=k, bias=b, out=out)
    ref = (a.double() @ w.double().T + b.double())
    err = (out.double() - ref).abs().max().item()
    scale = ref.abs().max().item()
    # fp32 SIMT kernel on the same inputs: the error an fp32 GEMM makes anyway
    simt = torch.zeros(m, n, device=dev)
    TK.gemm(a, w, m=m, k=k, bias=b, out=simt)
    simt_err = (simt.double() - ref).abs().max().item()
    assert err <= max(8 * simt_err, 1e-5 * max(1.0, scale)), (err, simt_err, scale)


def test_tc_lstm_epilogue_matches_simt():
    from paper_1909_08723_b200 import kernels as K
    dev = torch.device("cuda")
    torch.manual_seed(3)
    m, H, k = 333, 320, 1024
    a = torch.randn(m, k, device=dev) * 0.3
    w = _bf16_exact(torch.rand(4 * H, k, device=dev) * 0.1 - 0.05)
    b = torch.randn(4 * H, device=dev) * 0.1
    rows = torch.randperm(m, device=dev).to(torch.int32)
    parent = torch.randperm(m, device=dev).to(torch.int32)
    c_in = torch.randn(m, H, device=dev)
    h_res = torch.randn(m, H, device=dev)
    outs = []
    for tc in (False, True):
        c_out = torch.zeros(m, H, device=dev)
        h_out = torch.zeros(m, H, device=dev)
        kw = dict(m=m, k=k, bias=b, mode=1, hidden=H, rows=rows, parent=parent, c_in=c_in,
                  c_out=c_out, h_out=h_out, h_res=h_res)
        if tc:
            K.gemm_tc(_packed(a, k), _w(w), **kw)
        else:
            TK.gemm(a, w, **kw)
        outs.append((h_out, c_out))
    assert (outs[0][0] - outs[1][0]).abs().max().item() < 1e-5
    assert (outs[0][1] - outs[1][1]).abs().max().item() < 1e-5


def test_tc_device_row_count():
    """Rows past the device-side count are not written."""
    from paper_1909_08723_b200 import kernels as K
    dev = torch.device("cuda")
    m, n, k = 256, 128, 128
    a = torch.randn(m, k, device=dev)
    w = _bf16_exact(torch.randn(n, k, device=dev) * 0.1)
    out = torch.full((m, n), 7.0, device=dev)
    cnt = torch.tensor([130], dtype=torch.int32, device=dev)
    K.gemm_tc(_packed(a, k), _w(w), m=m, m_dev=cnt, k=k, out=out)
    ref = a.double() @ w.double().T
    assert (out[:130].double() - ref[:130]).abs().max().item() < 1e-4
    assert (out[130:] == 7.0).all()


@pytest.mark.parametrize("m,vw,k", [(37, 9000, 128), (300, 65000, 1216)])
def test_row_stats_feed_g_rows_and_eos(m, vw, k):
    """LM-output GEMM tile statistics -> fb_stats_to_g == single-pass
    fb_logits_to_g (the second shape is the c2 word-LM output projection)."""
    from paper_1909_08723_b200 import kernels as K
    dev = torch.device("cuda")
    torch.manual_seed(11 + m)
    n = vw + 3
    a = torch.randn(m, k, device=dev)
    w = _bf16_exact(torch.randn(n, k, device=dev) * 0.3)
    b = torch.randn(n, device=dev) * 0.5
    logits = torch.empty(m, n, device=dev)
    stats = torch.empty(m, (n + 63) // 64, 4, device=dev)
    K.gemm_tc(_packed(a, k), _w(w), m=m, k=k, bias=b, out=logits,
              row_stats=stats, stats_vw=vw)
    ref = a.double() @ w.double().T + b.double()
    assert (logits.double() - ref).abs().max().item() < 1e-5 * max(1.0, ref.abs().max().item())
    g_ref = torch.empty(m, vw, dtype=torch.float64, device=dev)
    e_ref = torch.empty(m, dtype=torch.float64, device=dev)
    K.logits_to_g(logits, vw, n, m=m, g_pool=g_ref, eos_out=e_ref)
    g = torch.empty_like(g_ref)
    e = torch.empty_like(e_ref)
    seg = torch.empty(m, (vw + 4095) // 4096 + 2, dtype=torch.float64, device=dev)
    cnt = torch.tensor([m], dtype=torch.int32, device=dev)
    K.stats_to_g(logits, stats, vw, n, m=m, m_dev=cnt, g_pool=g, eos_out=e, seg_ws=seg)
    assert (g - g_ref).abs().max().item() < 1e-13
    assert (e - e_ref).abs().max().item() < 1e-5
    # single-word masses from g differences agree to fp64 resolution of g (~1 ulp of 1.0)
    p = torch.diff(g, dim=1, prepend=torch.zeros(m, 1, dtype=torch.float64, device=dev))
    p_ref = torch.diff(g_ref, dim=1, prepend=torch.zeros(m, 1, dtype=torch.float64, device=dev))
    assert (p - p_ref).abs().max().item() < 1e-14      # segmented vs sequential scan order
    # statistics from an eos-only pass reused by a gathered g-row pass: bit-identical
    stat = torch.empty(m, 2, dtype=torch.float64, device=dev)
    e_ev = torch.empty_like(e_ref)
    K.stats_to_g(logits, stats, vw, n, m=m, m_dev=cnt, eos_out=e_ev, stat_out=stat)
    assert torch.equal(e_ev, e)
    # the <eos> fusion-column update fused into that pass == fb_eos_fixup after it
    from paper_1909_08723_b200 import _lib
    fus0 = torch.randn(m + 1, 52, dtype=torch.float64, device=dev)
    fus_a, fus_b = fus0.clone(), fus0.clone()
    rows_ev = torch.randperm(m, device=dev).to(torch.int32)
    e_a = torch.empty_like(e_ref)
    K.stats_to_g(logits, stats, vw, n, m=m, m_dev=cnt, slots=rows_ev, eos_out=e_a, fus=fus_a,
                 fus_eos=7)
    e_b = torch.empty_like(e_ref)
    K.stats_to_g(logits, stats, vw, n, m=m, m_dev=cnt, slots=rows_ev, eos_out=e_b)
    _lib.call("fb_eos_fixup", m, _lib.ptr(cnt), _lib.ptr(rows_ev), _lib.ptr(e_b),
              _lib.ptr(fus_b), fus_b.stride(0), 7, _lib.stream_ptr())
    assert torch.equal(e_a, e_b) and torch.equal(fus_a, fus_b)
    src = torch.randperm(m, device=dev)[:20].to(torch.int32)
    slots = torch.arange(20, dtype=torch.int32, device=dev).flip(0).contiguous()
    c20 = torch.tensor([20], dtype=torch.int32, device=dev)
    g2, e2 = torch.zeros(20, vw, dtype=torch.float64, device=dev), torch.zeros(20, dtype=torch.float64, device=dev)
    g3, e3 = torch.zeros_like(g2), torch.zeros_like(e2)
    K.stats_to_g(logits, stats, vw, n, m=20, m_dev=c20, src_rows=src, slots=slots, g_pool=g2,
                 eos_out=e2, seg_ws=seg)
    K.stats_to_g(logits, stats, vw, n, m=20, m_dev=c20, src_rows=src, slots=slots, g_pool=g3,
                 eos_out=e3, seg_ws=seg, stat_in=stat)
    assert torch.equal(g2, g3) and torch.equal(e2, e3)


@pytest.mark.parametrize("m,n,k,m_dev", [(160, 4800, 2432, 150), (64, 1280, 1024, 64),
                                         (600, 4800, 2432, 9), (128, 256, 4096, 128),
                                         (600, 4800, 2432, 600)])
def test_tc_stream_k(m, n, k, m_dev):
    """Stream-K (tiles < SMs): same result as one CTA per tile within fp32
    rounding, bit-identical across repeats (partials summed in K order), the
    arrival counters left zeroed, rows past the device count untouched."""
    from paper_1909_08723_b200 import kernels as K
    torch.manual_seed(m + n + k)
    dev = torch.device("cuda")
    a = torch.randn(m, k, device=dev) * 0.5
    w = _w(_bf16_exact(torch.rand(n, k, device=dev) * 0.2 - 0.1))
    b = torch.randn(n, device=dev)
    ap = _packed(a, k)
    cnt = torch.tensor([m_dev], dtype=torch.int32, device=dev)
    sk = K.SplitK(dev)
    outs = []
    for use in (None, sk, sk):
        out = torch.full((m, n), 7.0, device=dev)
        K.gemm_tc(ap, w, m=m, m_dev=cnt, k=k, bias=b, out=out, splitk=use)
        outs.append(out)
    ref = a[:m_dev].double() @ (w.double() * w.fb_acc_scale * K.operand_format()[2]).T + \
        b.double()
    scale = ref.abs().max().item()
    assert (outs[1][:m_dev].double() - ref).abs().max().item() < 1e-5 * max(1.0, scale)
    assert (outs[1][:m_dev] - outs[0][:m_dev]).abs().max().item() < 1e-5 * max(1.0, scale)
    assert torch.equal(outs[1], outs[2])
    assert (outs[1][m_dev:] == 7.0).all()
    assert int(sk.cnt.abs().sum()) == 0
    # LSTM epilogue through stream-K
    H = n // 4
    c_in = torch.randn(m, H, device=dev)
    res = []
    for use in (None, sk):
        c_out = torch.zeros(m, H, device=dev)
        h_out = torch.zeros(m, H, device=dev)
        K.gemm_tc(ap, w, m=m, m_dev=cnt, k=k, bias=b, mode=1, hidden=H, c_in=c_in, c_out=c_out,
                  h_out=h_out, splitk=use)
        res.append((h_out, c_out))
    assert (res[0][0] - res[1][0]).abs().max().item() < 1e-5
    assert (res[0][1] - res[1][1]).abs().max().item() < 1e-5
    assert int(sk.cnt.abs().sum()) == 0


@pytest.mark.parametrize("m,n,k", [(300, 52, 640), (129, 64, 128), (70, 33, 256)])
def test_tc_fused_epilogues_match_separate_kernels(m, n, k):
    """out_logsoftmax == GEMM + fb_log_softmax_rows and out_exp2 == exp(2 x),
    bit for bit (same arithmetic), rows gathered through `rows`."""
    from paper_1909_08723_b200 import kernels as K
    torch.manual_seed(m + n)
    dev = torch.device("cuda")
    a = torch.randn(m, k, device=dev)
    w = _w(_bf16_exact(torch.randn(n, k, device=dev) * 0.1))
    b = torch.randn(n, device=dev)
    ap = _packed(a, k)
    rows = torch.randperm(m, device=dev).to(torch.int32)
    logits = torch.zeros(m, n, device=dev)
    K.gemm_tc(ap, w, m=m, k=k, bias=b, out=logits, rows=rows, kcb=1)
    ref = torch.zeros(m, n, device=dev)
    K.log_softmax_rows(logits, ref, n, m=m, rows=rows)
    fused = torch.zeros(m, n, device=dev)
    K.gemm_tc(ap, w, m=m, k=k, bias=b, out=fused, rows=rows, kcb=1, out_logsoftmax=True)
    assert torch.equal(fused, ref)
    e = torch.zeros(m, n, device=dev)
    K.gemm_tc(ap, w, m=m, k=k, bias=b, out=e, rows=rows, kcb=1, out_exp2=True)
    assert torch.equal(e, torch.exp(2.0 * logits)) or \
        (e - torch.exp(2.0 * logits)).abs().max().item() <= 1e-6 * e.abs().max().item()


@pytest.mark.parametrize("m", [64, 150, 333])
def test_tc_lstm_epilogue_tma_rows_in_order(m):
    """LSTM cell with rows in GEMM order (the word LM: c, h and the next GEMM's
    h planes leave by TMA tensor stores) == the SIMT kernel, planes exact."""
    from paper_1909_08723_b200 import kernels as K
    dev = torch.device("cuda")
    torch.manual_seed(m)
    H, k = 1200, 2432
    a = torch.randn(m, k, device=dev) * 0.3
    w = _bf16_exact(torch.rand(4 * H, k, device=dev) * 0.1 - 0.05)
    b = torch.randn(4 * H, device=dev) * 0.1
    parent = torch.randperm(m, device=dev).to(torch.int32)
    c_in = torch.randn(m, H, device=dev)
    outs = []
    for tc in (False, True):
        c_out = torch.full((m, H), 7.0, device=dev)
        h_out = torch.full((m, H), 7.0, device=dev)
        kw = dict(m=m, k=k, bias=b, mode=1, hidden=H, parent=parent, c_in=c_in, c_out=c_out,
                  h_out=h_out)
        if tc:
            hs = K.operand_planes(m + 16, 1216, dev).zero_()
            K.gemm_tc(_packed(a, k), _w(w), h_split=hs, hs_by_row=True, **kw)
        else:
            TK.gemm(a, w, **kw)
        outs.append((h_out, c_out))
    assert (outs[0][0] - outs[1][0]).abs().max().item() < 1e-5
    assert (outs[0][1] - outs[1][1]).abs().max().item() < 1e-5
    h = outs[1][0]
    for q, ref_q in enumerate(_split_ref(h)):
        assert torch.equal(hs[q, :m, :H], ref_q)
    assert (hs[:, m:, :] == 0).all() and (hs[:, :, H:] == 0).all()


@pytest.mark.parametrize("n,k", [(4800, 2432), (1280, 320)])
def test_tc_few_tile_width_is_bit_identical(n, k):
    """Grids under a third of the SMs take 64-wide tiles (gemm_tc.cu): the
    first 64 rows of a 64-row GEMM (64-wide tiles) and of a 600-row GEMM
    (128-wide tiles) over the same operands are bit-identical, plain and
    LSTM-cell epilogues."""
    from paper_1909_08723_b200 import kernels as K
    dev = torch.device("cuda")
    torch.manual_seed(n + k)
    a = torch.randn(600, k, device=dev) * 0.3
    w = _w(_bf16_exact(torch.rand(n, k, device=dev) * 0.1 - 0.05))
    b = torch.randn(n, device=dev) * 0.1
    H = n // 4
    c_in = torch.randn(600, H, device=dev)
    res = {}
    for m in (64, 600):
        ap = _packed(a[:m], k)
        out = torch.empty(m, n, device=dev)
        K.gemm_tc(ap, w, m=m, k=k, bias=b, out=out)
        c_out = torch.empty(m, H, device=dev)
        h_out = torch.empty(m, H, device=dev)
        K.gemm_tc(ap, w, m=m, k=k, bias=b, mode=1, hidden=H, c_in=c_in[:m], c_out=c_out,
                  h_out=h_out)
        res[m] = (out, c_out, h_out)
    for x64, x600 in zip(res[64], res[600]):
        assert torch.equal(x64, x600[:64])

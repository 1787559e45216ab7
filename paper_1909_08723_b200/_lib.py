"""ctypes binding of the in-tree C-ABI library ``libfusedbeam_b200.so``.

The product path has no CPU fallback: every entry point raises when the
library is missing or was built for another architecture.  Status codes map to
the reference's exception types (``errors.py:4-13``): FB_ERR_VALUE ->
ValueError, FB_ERR_CONFIG -> ConfigError, FB_ERR_CUDA -> RuntimeError.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import ConfigError, FormatError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfusedbeam_b200.so")
if os.environ.get("FB_LIB_AB"):          # dev: A/B timing against another in-tree build
    LIB_PATH = os.path.join(_HERE, os.environ["FB_LIB_AB"])

i32, i64, f64, vp = C.c_int32, C.c_int64, C.c_double, C.c_void_p


class FbTrie(C.Structure):
    _fields_ = [("row_ptr", vp), ("edge_label", vp), ("edge_child", vp), ("info", vp),
                ("num_states", i32), ("num_words", i32), ("alphabet", i32)]


class FbSearchCfg(C.Structure):
    _fields_ = [("beam", i32), ("vocab", i32), ("pad_id", i32), ("eos_id", i32),
                ("cov_mode", i32), ("gate_on", i32), ("early_stop", i32), ("has_fusion", i32),
                ("am_f32", i32), ("max_tokens", i32), ("t_max", i32), ("pad0", i32),
                ("lm_weight", f64), ("cov_weight", f64), ("tau1", f64), ("tau2", f64),
                ("cov_margin", f64), ("gamma", f64)]


class FbSearchState(C.Structure):
    _fields_ = [(n, vp) for n in (
        "active", "n_live", "steps", "max_len", "t_enc",
        "base_in", "base_out", "total_in", "total_out", "tok_in", "tok_out",
        "parent", "last_tok", "acc_post", "cov_post",
        "fin_valid", "fin_total", "fin_len", "fin_tokens", "fin_acc",
        "res_len", "res_score", "res_finished", "res_steps", "res_tokens", "res_acc",
        "next_rows", "next_count", "cand_score_ws", "cand_flat_ws")] + [
        ("force_two_stage", i32), ("pad1", i32), ("fus_norm", vp), ("fus_floor", C.c_double),
        ("next_row_pos", vp), ("select_arrive", vp)]


class FbGemm(C.Structure):
    _fields_ = [("m_max", i32), ("m_dev", vp), ("n", i32), ("k", i32),
                ("a", vp), ("lda", i64), ("w", vp), ("ldw", i64), ("bias", vp),
                ("c", vp), ("ldc", i64), ("mode", i32), ("hidden", i32),
                ("rows", vp), ("parent", vp), ("c_in", vp), ("ld_cin", i64),
                ("c_out", vp), ("ld_cout", i64), ("h_out", vp), ("ld_h", i64),
                ("h_res", vp), ("ld_res", i64), ("addend", vp), ("ld_add", i64),
                ("h_split", vp), ("hs_plane_rows", i64), ("ld_hs", i64),
                ("row_stats", vp), ("stats_vw", i32), ("kcb", i32),
                ("hs_row_mode", i32), ("splitk_ws", vp), ("splitk_cnt", vp),
                ("out_exp2", i32), ("out_logsoftmax", i32), ("acc_scale", C.c_float),
                ("pad_fmt", i32)]


class FbSeg(C.Structure):
    _fields_ = [("src", vp), ("ld", i64), ("width", i32), ("mode", i32)]


class FbPack(C.Structure):
    _fields_ = [("seg", FbSeg * 4), ("nseg", i32), ("k_pad", i32), ("tok_default", i32),
                ("out_mode", i32), ("plane_rows", i64)]


_SIGS = {
    "fb_last_error": (C.c_char_p, []),
    "fb_abi_version": (C.c_int, []),
    "fb_launch_count": (C.c_ulonglong, []),
    "fb_launch_reset": (None, []),
    "fb_lookahead_scores": (C.c_int, [C.POINTER(FbTrie), i32, vp, vp, vp, vp, vp, i64, vp, vp,
                                      i32, i32, f64, f64, vp, i64, vp, vp]),
    "fb_trie_advance": (C.c_int, [C.POINTER(FbTrie), i32, vp, vp, vp, vp, vp, vp, i32, i32, i32,
                                  vp, vp, vp, vp]),
    "fb_cumsum_rows": (C.c_int, [i32, vp, i64, i32, vp, vp, i64, vp]),
    "fb_logits_to_g": (C.c_int, [i32, vp, vp, i64, vp, i32, i32, vp, vp, i64, vp, vp]),
    "fb_search_init": (C.c_int, [C.POINTER(FbSearchCfg), C.POINTER(FbSearchState), i32, vp]),
    "fb_search_step": (C.c_int, [C.POINTER(FbSearchCfg), C.POINTER(FbSearchState), i32, vp, i64,
                                 vp, i64, vp]),
    "fb_attend_coverage": (C.c_int, [C.POINTER(FbSearchCfg), i32, vp, vp, vp, vp, vp, vp, i32,
                                     i64, vp, vp, vp]),
    "fb_gather_rows": (C.c_int, [i32, vp, vp, vp, i64, vp]),
    "fb_gemm_tc": (C.c_int, [C.POINTER(FbGemm), i32, i64, vp]),
    "fb_stats_to_g": (C.c_int, [i32, vp, vp, i64, vp, i32, vp, i32, vp, vp, i64, vp, vp, vp, vp,
                                vp, i64, i32, vp]),
    "fb_lstm_recurrence": (C.c_int, [i32, i32, i32, vp, i32, vp, i64, i64, vp, i64, i64, vp,
                                      vp, C.c_float, vp, vp]),
    "fb_operand_format": (C.c_int, [vp, vp, vp]),
    "fb_pack_rows": (C.c_int, [C.POINTER(FbPack), i32, vp, vp, vp, vp, vp, vp, i64, vp]),
    "fb_log_softmax_rows": (C.c_int, [i32, vp, vp, vp, i64, i32, vp, i64, vp]),
    "fb_row_logsumexp": (C.c_int, [i32, vp, vp, vp, i64, i32, i32, vp, vp]),
    "fb_set_attention_tiling": (C.c_int, [i32, i32, i32]),
    "fb_attention_step": (C.c_int, [C.POINTER(FbSearchCfg), i32, vp, vp, vp, vp, vp, i32, i32,
                                    vp, vp, i64, vp, vp, vp, vp, vp, i64, vp, i64, vp, vp, i32,
                                    vp, i64, i64, vp, vp]),
    "fb_spec_events": (C.c_int, [C.POINTER(FbTrie), i32, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                 vp]),
    "fb_boundary_plan": (C.c_int, [i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, i32, vp, vp, vp, vp,
                                   vp, vp, vp, vp, vp, i32, vp]),
    "fb_spec_select": (C.c_int, [C.POINTER(FbSearchCfg), C.POINTER(FbSearchState), i32,
                                 C.POINTER(FbTrie), vp, vp, vp, i64, vp, i64, vp, vp, vp, vp, vp,
                                 vp, vp]),
    "fb_eos_fixup": (C.c_int, [i32, vp, vp, vp, vp, i64, i32, vp]),
    "fb_copy_rows": (C.c_int, [i32, vp, vp, vp, vp, vp, i64, vp]),
    "fb_exp2x": (C.c_int, [i64, vp, vp, vp]),
    "fb_multilevel_rows": (C.c_int, [C.POINTER(FbTrie), i32, vp, vp, vp, i64, vp, i32, i32,
                                     C.c_double, C.c_double, vp, i64, vp]),
    "fb_multilevel_advance": (C.c_int, [C.POINTER(FbTrie), i32, vp, vp, vp, vp, i64, i32, i32,
                                        i32, vp, vp, vp, vp, vp]),
    "fb_ark_read_matrix": (C.c_int, [C.c_char_p, i64, vp, i64, vp, vp]),
    "fb_host_copy_batch": (C.c_int, [i32, vp, vp, vp, i32]),
    "fb_ark_read_batch": (C.c_int, [i32, vp, vp, vp, vp, vp, vp, vp, i32]),
    "fb_pta1_read_header": (C.c_int, [C.c_char_p, vp, vp, vp, vp]),
    "fb_pta1_read": (C.c_int, [C.c_char_p, vp, vp, vp, vp, vp, vp]),
    "fb_pta1_write": (C.c_int, [C.c_char_p, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp]),
    "fb_trie_build_sizes": (C.c_int, [i32, vp, vp, i32, vp, vp]),
    "fb_trie_build": (C.c_int, [i32, vp, vp, i32, i32, i32, vp, vp, vp, vp, vp, vp]),
    "fb_keys_exp2t": (C.c_int, [i32, i32, i32, vp, vp, vp]),
    "fb_scp_parse": (C.c_int, [C.c_char_p, i64, C.c_char_p, i64, vp, vp, vp, vp]),
    "fb_ark_append_matrix": (C.c_int, [C.c_char_p, C.c_char_p, C.c_char_p, vp, i32, i32, vp]),
}

_OPTIONAL = {}
_lock = threading.Lock()
_lib = None


def lib():
    """Load (once) and return the library; raise loudly if it is unusable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"CUDA library {LIB_PATH} is missing: run "
                "`python -m paper_1909_08723_b200.csrc.build` (there is no CPU fallback)")
        handle = C.CDLL(LIB_PATH)
        for name, (res, args) in list(_SIGS.items()) + list(_OPTIONAL.items()):
            fn = getattr(handle, name, None)
            if fn is None:
                if name in _OPTIONAL:
                    continue
                raise RuntimeError(f"{LIB_PATH} does not export {name}")
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def register(name: str, restype, argtypes) -> None:
    """Declare an additional exported symbol (used by sibling modules)."""
    _SIGS[name] = (restype, argtypes)
    if _lib is not None:
        fn = getattr(_lib, name)
        fn.restype = restype
        fn.argtypes = argtypes


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().fb_last_error().decode(errors="replace")
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise ConfigError(msg)
    if rc == 4:
        raise FormatError(msg)
    if rc == 5:
        raise IOError(msg)
    raise RuntimeError(f"CUDA error: {msg}")


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def ptr(t) -> int:
    """Device pointer of a torch tensor (or 0 for None)."""
    return 0 if t is None else int(t.data_ptr())


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)

"""Seeded synthetic inputs: token set, lexicon, fbank features and random-init
weights for the BASELINE.json configurations.

Everything here is input data, not compute: the same arrays feed the CUDA path
and the CPU oracle.  Weights are drawn uniform(-s, s) and rounded to bf16 so
that a bf16 tensor-core operand holds them exactly ("GEMM
precision"); biases are fp32-exact as drawn.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, asdict
from typing import Dict, List, Optional, Tuple

import numpy as np

# WSJ character set (PAPER.md:280 footnote): 45 characters + 3 atomic symbols
# + 4 specials = 52.  Multi-character tokens can never be trie edges
# (lexicon_trie.py:27-39).
WSJ_CHARS = list("abcdefghijklmnopqrstuvwxyz") + list("0123456789") + \
    list("'.-&/_~!?")
WSJ_ATOMS = ["<*IN*>", "<*MR.*>", "<NOISE>"]

# English-ish letter frequencies for the synthetic lexicon.
_LETTER_FREQ = np.array([8.2, 1.5, 2.8, 4.3, 12.7, 2.2, 2.0, 6.1, 7.0, 0.15, 0.77,
                         4.0, 2.4, 6.7, 7.5, 1.9, 0.1, 6.0, 6.3, 9.1, 2.8, 0.98,
                         2.4, 0.15, 2.0, 0.074])


def wsj_token_list() -> List[str]:
    """File tokens; TokenDictionary adds <pad>,<eos>,<unk> and <space> -> 52."""
    return WSJ_CHARS + WSJ_ATOMS


def synth_lexicon(n_words: int, seed: int, mean_len: float = 6.5,
                  letters: str = "abcdefghijklmnopqrstuvwxyz") -> List[str]:
    """Distinct English-like words: Poisson(mean_len) lengths (>= 1), letters
    drawn from unigram frequencies; a small share carry an apostrophe."""
    rng = np.random.default_rng(seed)
    p = _LETTER_FREQ[:len(letters)] / _LETTER_FREQ[:len(letters)].sum()
    alphabet = np.array(list(letters))
    words = set()
    while len(words) < n_words:
        k = n_words - len(words)
        lens = np.maximum(1, rng.poisson(mean_len, size=k))
        for L in lens:
            w = "".join(rng.choice(alphabet, size=int(L), p=p))
            if L > 3 and rng.random() < 0.02:
                w = w[:-1] + "'" + w[-1]
            words.add(w)
            if len(words) == n_words:
                break
    return sorted(words)


def synth_fbank(n_utts: int, seed: int, frames: Tuple[int, int], feat_dim: int = 80,
                sort_by_length: bool = False) -> List[Tuple[str, np.ndarray]]:
    """[T, feat_dim] float32 N(0,1) per utterance, T ~ U{frames[0]..frames[1]}."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(frames[0], frames[1] + 1, size=n_utts)
    out = []
    for i, T in enumerate(lens):
        r = np.random.default_rng(seed * 1_000_003 + i)
        out.append((f"utt{i:05d}", r.standard_normal((int(T), feat_dim)).astype(np.float32)))
    if sort_by_length:
        out.sort(key=lambda u: (u[1].shape[0], u[0]))
    return out


@dataclass
class AsrDims:
    feat_dim: int = 80
    subsample: int = 4
    enc_layers: int = 4
    enc_hidden: int = 320          # per direction; encoder output C = 2 * enc_hidden
    dec_layers: int = 3
    dec_hidden: int = 320
    emb: int = 48
    att: int = 320
    vocab: int = 52
    out_scale: float = 0.35        # uniform range of the output projection
    eos_bias: float = 0.0          # added to the <eos> output bias

    @property
    def ctx(self) -> int:
        return 2 * self.enc_hidden


@dataclass
class LmDims:
    layers: int = 3
    hidden: int = 1200             # == embedding dim (tied input/output)
    words: int = 65000             # closed vocabulary; outputs = words + 3
    emb_scale: float = 0.08
    eos_bias: float = 7.0          # </s> output bias (sentence-length prior)
    w_scale: float = 1.0           # LSTM weight range multiplier (x 1/sqrt(hidden))


@dataclass
class SubwordLmDims:
    """Token-level (subword) LSTM LM for SubwordFusion (config 4)."""
    layers: int = 4
    hidden: int = 800
    emb: int = 800
    vocab: int = 5000              # == the token dictionary size
    out_scale: float = 0.25        # uniform range of the output projection
    eos_bias: float = 0.0          # added to the <eos> output bias
    w_scale: float = 1.0


def subword_token_list(n_tokens: int, seed: int) -> List[str]:
    """Distinct synthetic subword strings (1-4 letters, word-initial ones
    marked with a leading '_'); TokenDictionary adds the 4 specials."""
    rng = np.random.default_rng(seed)
    p = _LETTER_FREQ / _LETTER_FREQ.sum()
    alphabet = np.array(list("abcdefghijklmnopqrstuvwxyz"))
    toks: List[str] = []
    seen = set()
    while len(toks) < n_tokens:
        L = int(rng.integers(1, 5))
        t = ("_" if rng.random() < 0.4 else "") + "".join(rng.choice(alphabet, size=L, p=p))
        if t not in seen:
            seen.add(t)
            toks.append(t)
    return toks


def _bf16_round(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bf16, returned as fp32 (exact in bf16)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def _uniform(rng, shape, s) -> np.ndarray:
    return _bf16_round(rng.uniform(-s, s, size=shape).astype(np.float32))


def asr_weights(d: AsrDims, seed: int, eos_id: int = 1) -> Dict[str, np.ndarray]:
    """Encoder + attention-LSTM decoder weights."""
    rng = np.random.default_rng(seed)
    W: Dict[str, np.ndarray] = {}
    He = d.enc_hidden
    se = 1.0 / math.sqrt(He)
    for l in range(d.enc_layers):
        fin = d.feat_dim * d.subsample if l == 0 else 2 * He
        for dr in range(2):
            W[f"enc.{l}.{dr}.w_ih"] = _uniform(rng, (4 * He, fin), se)
            W[f"enc.{l}.{dr}.w_hh"] = _uniform(rng, (4 * He, He), se)
            W[f"enc.{l}.{dr}.b"] = _uniform(rng, (4 * He,), se)
    H, C = d.dec_hidden, d.ctx
    sd = 1.0 / math.sqrt(H)
    W["dec.emb"] = _uniform(rng, (d.vocab, d.emb), 1.0)
    for l in range(d.dec_layers):
        fin = (d.emb + C) if l == 0 else (H + C)
        W[f"dec.{l}.w_ih"] = _uniform(rng, (4 * H, fin), sd)
        W[f"dec.{l}.w_hh"] = _uniform(rng, (4 * H, H), sd)
        W[f"dec.{l}.b"] = _uniform(rng, (4 * H,), sd)
    W["dec.att.w_k"] = _uniform(rng, (d.att, C), 1.0 / math.sqrt(C))
    W["dec.att.b_k"] = _uniform(rng, (d.att,), 1.0 / math.sqrt(C))
    W["dec.att.w_q"] = _uniform(rng, (d.att, H), sd)
    W["dec.att.v"] = _uniform(rng, (d.att,), 1.0)
    W["dec.out.w"] = _uniform(rng, (d.vocab, H + C), d.out_scale)
    b = _uniform(rng, (d.vocab,), d.out_scale)
    b[eos_id] = _bf16_round(np.array([b[eos_id] + d.eos_bias], np.float32))[0]
    W["dec.out.b"] = b
    return W


def lm_weights(d: LmDims, seed: int) -> Dict[str, np.ndarray]:
    """Tied-embedding LSTM word LM (outputs: words, </s>, <unk>, <s>)."""
    rng = np.random.default_rng(seed)
    H = d.hidden
    s = d.w_scale / math.sqrt(H)
    W: Dict[str, np.ndarray] = {}
    W["lm.emb"] = _uniform(rng, (d.words + 3, H), d.emb_scale)
    for l in range(d.layers):
        W[f"lm.{l}.w_ih"] = _uniform(rng, (4 * H, H), s)
        W[f"lm.{l}.w_hh"] = _uniform(rng, (4 * H, H), s)
        W[f"lm.{l}.b"] = _uniform(rng, (4 * H,), s)
    b = _uniform(rng, (d.words + 3,), 0.5)
    b[d.words] = _bf16_round(np.array([d.eos_bias], np.float32))[0]
    W["lm.b_out"] = b
    return W


def subword_lm_weights(d: SubwordLmDims, seed: int, eos_id: int = 1) -> Dict[str, np.ndarray]:
    """Token-level LSTM LM: embedding, L LSTM layers, untied output projection."""
    rng = np.random.default_rng(seed)
    H, E = d.hidden, d.emb
    s = d.w_scale / math.sqrt(H)
    W: Dict[str, np.ndarray] = {}
    W["slm.emb"] = _uniform(rng, (d.vocab, E), 1.0)
    for l in range(d.layers):
        W[f"slm.{l}.w_ih"] = _uniform(rng, (4 * H, E if l == 0 else H), s)
        W[f"slm.{l}.w_hh"] = _uniform(rng, (4 * H, H), s)
        W[f"slm.{l}.b"] = _uniform(rng, (4 * H,), s)
    W["slm.out.w"] = _uniform(rng, (d.vocab, H), d.out_scale)
    b = _uniform(rng, (d.vocab,), d.out_scale)
    b[eos_id] = _bf16_round(np.array([b[eos_id] + d.eos_bias], np.float32))[0]
    W["slm.out.b"] = b
    return W


@dataclass
class Workload:
    """One BASELINE.json configuration."""
    name: str
    n_utts: int
    frames: Tuple[int, int]
    beam: int
    asr: AsrDims
    lm: Optional[LmDims]
    lm_weight: float = 0.0
    coverage_mode: str = "off"
    coverage_weight: float = 0.01
    eos_gamma: Optional[float] = None
    max_len_ratio: float = 1.0
    batch_size: int = 512
    seed: int = 1234
    sublm: Optional[SubwordLmDims] = None      # SubwordFusion (config 4) instead of look-ahead

    def describe(self) -> dict:
        out = asdict(self)
        out["frames"] = list(self.frames)
        return out


# eos_bias 0.5 (scripts/calib.sh): c3 (coverage + EOS gate) finishes ~40% of its
# utterances after ~45 steps; c1 (no gate) decodes to its length cap
SMALL_ASR = AsrDims(enc_layers=2, enc_hidden=128, dec_layers=1, dec_hidden=128,
                    emb=32, att=128, out_scale=0.5, eos_bias=0.5)

WORKLOADS: Dict[str, Workload] = {
    # configs[0]: CPU-runnable reference case
    "c1": Workload("c1", 16, (300, 300), 5, SMALL_ASR, None, batch_size=16),
    # configs[1]: the headline (WSJ-shaped, beam 10, 65k look-ahead LSTM LM)
    # output/LM scales calibrated so the random model decodes WSJ-like lengths
    # (~100 steps, ~3/4 of utterances emit <eos>; bench.py --stats)
    "c2": Workload("c2", 512, (700, 900), 10, AsrDims(out_scale=0.7),
                   LmDims(emb_scale=0.2, eos_bias=5.0, w_scale=2.0), lm_weight=0.5,
                   batch_size=512),
    "c3": Workload("c3", 16, (300, 300), 20, SMALL_ASR, None, coverage_mode="improved",
                   coverage_weight=0.01, eos_gamma=1.5, batch_size=16),
    # c4: subword decoder (5k tokens), beam 60, token-level LSTM-LM shallow fusion;
    # scales calibrated like c2 (scripts/calib_c4.sh: ~0.45 tokens per encoder
    # frame, ~60% of utterances emit <eos>, distinct outputs); batches of 256
    # (1.9x the throughput of 32 on a B200, same results: batch invariance)
    "c4": Workload("c4", 2620, (300, 3500), 60,
                   AsrDims(enc_hidden=512, dec_hidden=1024, emb=256, att=512, vocab=5000,
                           out_scale=1.5, eos_bias=1.0),
                   None, lm_weight=0.3, batch_size=256,
                   sublm=SubwordLmDims(layers=4, hidden=800, emb=800, vocab=5000,
                                       out_scale=0.5)),
    # c5: Switchboard-shaped char decoder, 30k-word look-ahead, beam 35.
    # The random model is bimodal in <eos> (scripts/calib.sh, 128 utts): a
    # higher eos bias ends every decode at step 2, this one decodes close to
    # the length cap (~9% finish, ~96% of T_enc steps, 115/128 distinct
    # outputs) -- full beams, word boundaries and LM events throughout.
    "c5": Workload("c5", 4458, (100, 2000), 35,
                   AsrDims(enc_hidden=320, dec_hidden=640, emb=64, att=320, out_scale=1.5,
                           eos_bias=-2.0),
                   LmDims(layers=3, hidden=1800 // 2, words=30000, emb_scale=0.2, eos_bias=5.0,
                          w_scale=2.0), lm_weight=0.25, batch_size=256),
}

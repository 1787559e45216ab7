"""Oracle restatement of the batched beam search (``decoder.py``).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Follows ``decoder.py:36-61`` (coverage, EOS gate), ``decoder.py:64-106``
(config), ``decoder.py:322-323`` (finished-set key) and the lock-step loop of
``decoder.py:339-480`` plus ``decode_corpus`` ``decoder.py:483-504``.  Scores are
float64 with the reference's operation order, so this restatement reproduces
the reference bit-for-bit (pinned by ``tests/golden``).

Extra (not in the reference): ``margins`` -- per utterance, the smallest score
gap that decided anything (adjacent candidates around and inside the beam cut,
the early-stop comparison, the finished-set cap and the final pick).  A GPU run
whose fp32 model arithmetic differs from this CPU run by less than that gap
must reproduce the same tokens; the parity tests use it to exempt genuine
near-ties, as ``BASELINE.json.north_star`` allows.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

NEG_INF = float("-inf")


def cov_original(acc, tau1: float) -> float:
    """decoder.py:36-38 (Eq. 5): frames with accumulated attention > tau1."""
    return float(np.count_nonzero(np.asarray(acc) > tau1))


def cov_improved(acc, tau1: float, tau2: float, margin: float) -> float:
    """decoder.py:41-48 (Eq. 6): count above tau1 minus (c + acc - tau2) above tau2.
    The penalty is a numpy (pairwise) sum over all frames, zeros included."""
    a = np.asarray(acc, dtype=np.float64)
    n_att = np.count_nonzero(a > tau1)
    pen = np.where(a > tau2, margin + a - tau2, 0.0).sum()
    return float(n_att - pen)


def eos_ok(row, gamma: Optional[float], eos_id: int) -> bool:
    """decoder.py:51-61 (Eq. 7): log P(eos) > gamma * max_t log P(t); None = off."""
    if gamma is None:
        return True
    r = np.asarray(row)
    return bool(r[eos_id] > gamma * r.max())


@dataclass
class OracleConfig:
    """decoder.py:64-106."""
    beam_size: int = 50
    lm_weight: float = 0.9
    coverage_mode: str = "off"
    coverage_weight: float = 0.01
    tau1: float = 0.5
    tau2: float = 1.0
    cov_margin: float = 0.7
    eos_gamma: Optional[float] = None
    max_len_ratio: float = 1.0

    def coverage(self, acc) -> float:
        if self.coverage_mode == "original":
            return cov_original(acc, self.tau1)
        if self.coverage_mode == "improved":
            return cov_improved(acc, self.tau1, self.tau2, self.cov_margin)
        return 0.0


@dataclass
class OracleResult:
    utt_id: str
    tokens: List[int]
    score: float
    attn_accum: np.ndarray
    finished: bool
    steps: int
    margin: float = math.inf          # smallest deciding gap (see module doc)
    decision_margin: float = math.inf  # same, without the in-beam order gaps


@dataclass
class _H:
    toks: Tuple[int, ...]
    base: float
    total: float
    acc: np.ndarray


def _key(h: _H):
    return (-h.total, len(h.toks), h.toks)       # decoder.py:322-323


@dataclass
class _U:
    uid: str
    am: object
    t_enc: int
    max_len: int
    live: List[_H]
    done: List[_H] = field(default_factory=list)
    last: List[int] = field(default_factory=lambda: [-1])
    on: bool = True
    steps: int = 0
    margin: float = math.inf
    dmargin: float = math.inf


def _gap(a: float, b: float) -> float:
    if a == b:
        return 0.0
    if math.isinf(a) or math.isinf(b):
        return math.inf
    return abs(a - b)


def decode_batch(features, scorer, fusion, cfg: OracleConfig, d) -> List[OracleResult]:
    """decoder.py:339-480 restated.  ``features`` are objects with ``utt_id`` and
    ``data``; ``scorer`` implements init/enc_length/step/reorder; ``fusion`` is
    None or implements start/char_scores/advance/reorder/nonpositive_scores."""
    V = len(d)
    eos, pad = d.eos_id, d.pad_id
    cov_on = cfg.coverage_mode != "off"
    early = fusion is None or fusion.nonpositive_scores
    utts: List[_U] = []
    for f in features:
        if np.asarray(f.data).size == 0:
            raise ValueError(f"utterance {f.utt_id!r}: empty feature matrix")
        st = scorer.init(f)
        T = scorer.enc_length(st)
        utts.append(_U(f.utt_id, st, T, max(1, int(math.floor(cfg.max_len_ratio * T))),
                       [_H((), 0.0, 0.0, np.zeros(T))]))
    fst = fusion.start(len(utts)) if fusion is not None else None

    while any(u.on for u in utts):
        act = [u for u in utts if u.on]
        frows = None
        base_row: Dict[int, int] = {}
        if fusion is not None:
            pos = 0
            for i, u in enumerate(act):
                base_row[i] = pos
                pos += len(u.live)
            frows = fusion.char_scores(fst)
            if frows.shape != (pos, V):
                raise ValueError("fusion scorer returned a bad shape")
        nxt_par: List[int] = []
        nxt_tok: List[int] = []
        for i, u in enumerate(act):
            n = len(u.live)
            am, attn, u.am = scorer.step(u.am, u.last)
            if am.shape != (n, V):
                raise ValueError("acoustic scorer returned a bad shape")
            step = np.array(am, dtype=np.float64, copy=True)
            if fusion is not None:
                step += cfg.lm_weight * frows[base_row[i]:base_row[i] + n]
            step[:, pad] = NEG_INF
            if cfg.eos_gamma is not None:
                shut = am[:, eos] <= cfg.eos_gamma * am.max(axis=1)
                step[shut, eos] = NEG_INF
            tot = np.array([h.total for h in u.live])
            flat = (tot[:, None] + step).T.ravel()       # token-major (decoder.py:404)
            order = np.argsort(-flat, kind="stable")
            keep: List[_H] = []
            par: List[int] = []
            tok_out: List[int] = []
            took = 0
            for j in order:
                sc = flat[j]
                if sc == NEG_INF or took == cfg.beam_size:
                    break
                took += 1
                t, p = int(j) // n, int(j) % n
                h = u.live[p]
                nb = h.base + float(step[p, t])
                acc = h.acc + attn[p]
                tt = nb + cfg.coverage_weight * cfg.coverage(acc) if cov_on else nb
                child = _H(h.toks + (t,), nb, tt, acc)
                if t == eos:
                    u.done.append(child)
                else:
                    keep.append(child)
                    par.append(p)
                    tok_out.append(t)
            # margins that decided the cut and the in-beam order
            srt = flat[order[:took + 1]]
            for a, b in zip(srt[:-1], srt[1:]):
                u.margin = min(u.margin, _gap(float(a), float(b)))
            # set membership only flips at the cut (the in-beam order decides
            # nothing but exact ties, which are themselves gaps of 0 at a cut)
            if 0 < took < len(order):
                u.dmargin = min(u.dmargin, _gap(float(flat[order[took - 1]]),
                                                float(flat[order[took]])))
            if len(u.done) > cfg.beam_size:
                u.done.sort(key=_key)
                cut = u.done[cfg.beam_size - 1].total, u.done[cfg.beam_size].total
                u.margin = min(u.margin, _gap(*cut))
                u.dmargin = min(u.dmargin, _gap(*cut))
                del u.done[cfg.beam_size:]
            u.steps += 1
            u.live = keep
            u.last = tok_out
            if not keep or u.steps >= u.max_len:
                u.on = False
            elif u.done and early:
                slack = cfg.coverage_weight * u.t_enc if cov_on else 0.0
                best = max(h.base for h in keep) + slack
                worst = min(h.total for h in u.done)
                u.margin = min(u.margin, _gap(best, worst))
                u.dmargin = min(u.dmargin, _gap(best, worst))
                if best < worst:
                    u.on = False
            if u.on:
                u.am = scorer.reorder(u.am, par)
                if fusion is not None:
                    nxt_par.extend(base_row[i] + p for p in par)
                    nxt_tok.extend(tok_out)
        if fusion is not None:
            fst = fusion.reorder(fst, nxt_par)
            if nxt_tok:
                fst = fusion.advance(fst, np.asarray(nxt_tok, dtype=np.int64))

    out = []
    for u in utts:
        pool = u.done if u.done else u.live
        if not pool:
            raise ValueError(f"utterance {u.uid!r}: no hypotheses survived decoding")
        ranked = sorted(pool, key=_key)
        if len(ranked) > 1:
            u.margin = min(u.margin, _gap(ranked[0].total, ranked[1].total))
            u.dmargin = min(u.dmargin, _gap(ranked[0].total, ranked[1].total))
        best = ranked[0]
        toks = list(best.toks)
        if toks and toks[-1] == eos:
            toks.pop()
        out.append(OracleResult(u.uid, toks, best.total, best.acc, bool(u.done),
                                u.steps, u.margin, u.dmargin))
    return out


def decode_corpus(features, scorer, fusion_factory, cfg: OracleConfig, d,
                  batch_size: int = 8) -> List[OracleResult]:
    """decoder.py:483-504 (sequential form): input-order chunks, one fusion per chunk."""
    res: List[OracleResult] = []
    for i in range(0, len(features), batch_size):
        fus = fusion_factory() if fusion_factory is not None else None
        res.extend(decode_batch(features[i:i + batch_size], scorer, fus, cfg, d))
    return res

"""CPU-side workload harness for the oracle -- TEST INFRASTRUCTURE ONLY.

Builds a BASELINE.json configuration's seeded inputs (the synthesizer
``paper_1909_08723_b200/synth.py`` loaded BY FILE PATH, so the product
package and its CUDA library are never imported), the oracle models over them,
and decodes utterances with the oracle restatement of the reference decoder
(``oracle/search.py`` <- ``decoder.py:339-480``) on a pool of worker processes,
one per host core, each single-threaded.

Users: ``bench.py`` (the ``--impl reference`` arm and the ``cpu_baseline``
leg), ``tests/golden/make_parity.py`` (full-set parity fixtures) and the parity
tests.  Never the product.
"""

from __future__ import annotations

import dataclasses
import importlib.util
import math
import multiprocessing as mp
import os
import sys
from multiprocessing.connection import wait
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_SYNTH = None


def synth():
    """``paper_1909_08723_b200/synth.py`` (pure numpy input generation) without
    running the product package's ``__init__``."""
    global _SYNTH
    if _SYNTH is None:
        mod = sys.modules.get("paper_1909_08723_b200.synth")
        if mod is None:
            path = os.path.join(ROOT, "paper_1909_08723_b200", "synth.py")
            spec = importlib.util.spec_from_file_location("_fb_synth_standalone", path)
            mod = importlib.util.module_from_spec(spec)
            sys.modules[spec.name] = mod          # dataclasses resolve their module
            spec.loader.exec_module(mod)
        _SYNTH = mod
    return _SYNTH


def workload(name: str, n_utts: Optional[int] = None, words: Optional[int] = None,
             overrides: Sequence[str] = ()):
    """WORKLOADS[name] with the bench's optional overrides (``part.field=value``)."""
    S = synth()
    wl = S.WORKLOADS[name]
    if n_utts is not None:
        wl = dataclasses.replace(wl, n_utts=n_utts, batch_size=min(wl.batch_size, n_utts))
    if words is not None and wl.lm is not None:
        wl = dataclasses.replace(wl, lm=dataclasses.replace(wl.lm, words=words))
    for ov in overrides:
        key, val = ov.split("=")
        part, field = key.split(".")
        if part == "wl":
            wl = dataclasses.replace(wl, **{field: type(getattr(wl, field))(val)})
        else:
            sub = getattr(wl, part)
            wl = dataclasses.replace(wl, **{part: dataclasses.replace(sub, **{field: float(val)})})
    return wl


def file_tokens(wl) -> List[str]:
    S = synth()
    if wl.sublm is not None:
        return S.subword_token_list(wl.asr.vocab - 4, seed=wl.seed + 3)
    return S.wsj_token_list()


def corpus(wl, rank: int = 0) -> List[Tuple[str, np.ndarray]]:
    """The rank's seeded, length-sorted utterances (same draw as bench.py)."""
    return synth().synth_fbank(wl.n_utts, seed=wl.seed + 100 + rank, frames=wl.frames,
                               feat_dim=wl.asr.feat_dim, sort_by_length=True)


class _Feat:
    def __init__(self, u, x):
        self.utt_id, self.data = u, x


class OracleModel:
    """Oracle scorer + fusion + config of one workload (weights from the seeded
    synthesizer, trie from the oracle's restated ``build_trie``)."""

    def __init__(self, wl, dtype=None):
        """dtype=torch.float64: every neural adapter in double precision (the
        exact-arithmetic yardstick for the fp32 oracle and the GPU)."""
        import torch  # (PyTorch-CPU fp32 adapters)
        dtype = dtype or torch.float32
        from .lexicon import OracleDict, build_trie
        from .neural import OracleAttnLstmScorer, OracleLstmWordLM
        from .search import OracleConfig
        S = synth()
        self.wl = wl
        self.d = od = OracleDict(file_tokens(wl))
        W = S.asr_weights(wl.asr, seed=wl.seed, eos_id=od.eos_id)
        self.lm = self.sublm = self.trie = None
        if wl.sublm is not None:
            from .subword import OracleLstmCharLM
            W.update(S.subword_lm_weights(wl.sublm, seed=wl.seed + 1, eos_id=od.eos_id))
            self.sublm = OracleLstmCharLM(W, wl.sublm.layers, od.pad_id, od.eos_id, dtype=dtype)
        if wl.lm is not None:
            W.update(S.lm_weights(wl.lm, seed=wl.seed + 1))
            self.words = S.synth_lexicon(wl.lm.words, seed=wl.seed + 2)
            self.trie = build_trie(self.words, od)
            self.lm = OracleLstmWordLM(W, wl.lm.layers, wl.lm.words, dtype=dtype)
        self.scorer = OracleAttnLstmScorer(W, wl.asr.enc_layers, wl.asr.dec_layers,
                                           wl.asr.subsample, od.eos_id, dtype=dtype)
        self.cfg = OracleConfig(beam_size=wl.beam, lm_weight=wl.lm_weight,
                                coverage_mode=wl.coverage_mode,
                                coverage_weight=wl.coverage_weight, eos_gamma=wl.eos_gamma,
                                max_len_ratio=wl.max_len_ratio)

    def fusion(self):
        """A fresh fusion per batch (decode_corpus, decoder.py:495-497)."""
        if self.sublm is not None:
            from .subword import OracleSubwordFusion
            return OracleSubwordFusion(self.sublm)
        if self.lm is not None:
            from .lookahead import OracleLookahead
            self.lm.clear_cache()             # bounded memory between utterances
            return OracleLookahead(self.trie, self.lm, self.d)
        return None

    def decode(self, utts: Sequence[Tuple[str, np.ndarray]]):
        from .search import decode_batch
        return decode_batch([_Feat(u, x) for u, x in utts], self.scorer, self.fusion(),
                            self.cfg, self.d)


# ---- one process per host core -------------------------------------------------
def _worker(conn, wl_args, rank, fp64=False):
    import torch
    torch.set_num_threads(1)
    wl = workload(*wl_args)
    model = OracleModel(wl, torch.float64 if fp64 else None)
    utts = corpus(wl, rank)
    conn.send(("ready", None))
    while True:
        msg = conn.recv()
        if msg is None:
            break
        i = int(msg)
        r = model.decode([utts[i]])[0]
        r.attn_accum = np.asarray(r.attn_accum, np.float64)
        conn.send(("done", (i, r)))
    conn.close()


def host_cores() -> int:
    return len(os.sched_getaffinity(0))


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class OraclePool:
    """``procs`` single-threaded worker processes, each holding the oracle
    model and the rank's corpus; ``decode(indices)`` hands utterances out
    longest-first to whichever worker is free (LPT) and returns results in
    the order of ``indices``."""

    def __init__(self, name: str, procs: Optional[int] = None, rank: int = 0,
                 n_utts: Optional[int] = None, words: Optional[int] = None,
                 overrides: Sequence[str] = (), fp64: bool = False):
        self.procs = procs or host_cores()
        self.wl = workload(name, n_utts, words, overrides)
        self.lengths = [x.shape[0] for _, x in corpus(self.wl, rank)]
        ctx = mp.get_context("spawn")
        self.conns, self.ps = [], []
        args = (name, n_utts, words, tuple(overrides))
        for _ in range(self.procs):
            a, b = ctx.Pipe()
            p = ctx.Process(target=_worker, args=(b, args, rank, fp64), daemon=True)
            p.start()
            self.conns.append(a)
            self.ps.append(p)
        for c in self.conns:
            assert c.recv()[0] == "ready"

    def decode(self, indices: Sequence[int]):
        todo = sorted(indices, key=lambda i: (-self.lengths[i], i))
        out: Dict[int, object] = {}
        free = list(self.conns)
        busy = set()
        while todo or busy:
            while todo and free:
                c = free.pop()
                c.send(todo.pop(0))
                busy.add(c)
            for c in wait(list(busy)):
                kind, (i, r) = c.recv()
                out[i] = r
                busy.discard(c)
                free.append(c)
        return [out[i] for i in indices]

    def close(self):
        for c in self.conns:
            try:
                c.send(None)
            except (BrokenPipeError, OSError):
                pass
        for p in self.ps:
            p.join(timeout=10)
            if p.is_alive():
                p.terminate()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def strata(n_utts: int, n: int) -> List[int]:
    """n indices evenly spaced over the length-sorted corpus (shortest to longest)."""
    n = max(1, min(n, n_utts))
    return sorted({int(round(x)) for x in np.linspace(0, n_utts - 1, n)})

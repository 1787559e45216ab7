"""Host-side data formats either side of the decode path,
read/written by the native C++ code (csrc/host_io.cu) and checked against files
and error behaviour recorded from the reference (tests/golden/formats/, made by
make_golden.py from lexicon_trie.py:178-224 and kaldi_io.py:44-160).  CPU only:
the library loads without a GPU and these entry points never touch one."""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import load_golden

FDIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "formats")


def m():
    import paper_1909_08723_b200 as fb
    return fb


def test_pta1_load_matches_reference_and_save_is_byte_identical(tmp_path):
    fb = m()
    from paper_1909_08723_b200.lexicon_trie import PrefixTreeAutomaton
    g = load_golden("formats.pkl.gz")
    for t in g["tries"]:
        src = os.path.join(FDIR, t["file"])
        trie = PrefixTreeAutomaton.load(src)
        np.testing.assert_array_equal(trie.transitions, t["transitions"])
        np.testing.assert_array_equal(trie.edge_labels, t["edge_labels"])
        np.testing.assert_array_equal(trie.is_final, t["is_final"])
        np.testing.assert_array_equal(trie.word_index, t["word_index"])
        np.testing.assert_array_equal(trie.ub_index, t["ub"])
        np.testing.assert_array_equal(trie.lb_index, t["lb"])
        out = tmp_path / t["file"]
        trie.save(str(out))
        assert out.read_bytes() == open(src, "rb").read()
        # the native builder produces the same automaton as the reference file
        built = fb.build_trie(t["words"], fb.TokenDictionary(t["letters"]))
        np.testing.assert_array_equal(built.transitions, t["transitions"])
        np.testing.assert_array_equal(built.lb_index, t["lb"])


def test_pta1_errors_match_reference():
    from paper_1909_08723_b200.errors import FormatError
    from paper_1909_08723_b200.lexicon_trie import PrefixTreeAutomaton
    g = load_golden("formats.pkl.gz")
    for name, (etype, msg) in g["pta_bad"].items():
        assert etype == "FormatError"
        with pytest.raises(FormatError) as ei:
            PrefixTreeAutomaton.load(os.path.join(FDIR, name))
        assert str(ei.value).endswith(msg.split(": ", 1)[1]), (name, str(ei.value), msg)


def test_scp_ark_reference_files(monkeypatch):
    from paper_1909_08723_b200 import kaldi_io as kio
    g = load_golden("formats.pkl.gz")
    monkeypatch.chdir(FDIR)
    entries = kio.read_scp("feats.scp")
    assert [e.utt_id for e in entries] == list(g["mats"])
    for e in entries:
        f = kio.read_feature(e)
        assert f.data.dtype == np.float32
        np.testing.assert_array_equal(f.data, g["mats"][e.utt_id])
    batch = kio.read_features_pinned(entries, threads=3)
    for f in batch:
        np.testing.assert_array_equal(f.data, g["mats"][f.utt_id])


def test_ark_and_scp_errors_match_reference(monkeypatch):
    from paper_1909_08723_b200 import kaldi_io as kio
    from paper_1909_08723_b200.errors import FormatError
    g = load_golden("formats.pkl.gz")
    monkeypatch.chdir(FDIR)
    types = {"FormatError": FormatError, "OSError": OSError}
    for name, (off, etype, msg) in g["ark_bad"].items():
        with pytest.raises(types[etype]) as ei:
            kio.read_ark_matrix(name, off)
        assert str(ei.value) == msg, (name, str(ei.value), msg)
        # the batch reader reports the same record error
        ok = kio.read_scp("feats.scp")[0]
        with pytest.raises(types[etype]) as ei:
            kio.read_features_pinned([ok, kio.ScpEntry("bad", name, off)])
        assert str(ei.value) == msg
    for name, (etype, msg) in g["scp_bad"].items():
        with pytest.raises(FormatError) as ei:
            kio.read_scp(name)
        assert str(ei.value) == msg


def test_ark_write_read_roundtrip(tmp_path):
    from paper_1909_08723_b200 import kaldi_io as kio
    rng = np.random.default_rng(3)
    ark, scp = str(tmp_path / "a.ark"), str(tmp_path / "a.scp")
    mats = {f"u{i}": rng.standard_normal((int(rng.integers(1, 50)), 80)).astype(np.float32)
            for i in range(6)}
    for u, x in mats.items():
        kio.write_ark_matrix(u, x, ark, scp)
    got = kio.read_features_pinned(kio.read_scp(scp), threads=4)
    for f in got:
        np.testing.assert_array_equal(f.data, mats[f.utt_id])
    with pytest.raises(ValueError):
        kio.write_ark_matrix("bad id", mats["u0"], ark, scp)


def test_native_build_trie_speed_and_equality():
    """The C++ sweep on a 65k-word lexicon equals the CSR invariants and is fast."""
    import time
    fb = m()
    from paper_1909_08723_b200 import synth
    d = fb.TokenDictionary(synth.wsj_token_list())
    words = synth.synth_lexicon(65000, seed=1236)
    t0 = time.perf_counter()
    trie = fb.build_trie(words, d)
    dt = time.perf_counter() - t0
    assert trie.num_words == 65000
    ranked = trie.words(d)
    assert ranked == sorted(words, key=lambda w: [d.index(c) for c in w])
    assert dt < 5.0, dt

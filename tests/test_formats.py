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


def test_scp_parser_matches_reference_cases(tmp_path):
    """The native SCP parser on line-ending / whitespace / int() edge cases and
    every error kind, against the reference read_scp's results and messages
    (tests/golden/make_scp_cases.py)."""
    from paper_1909_08723_b200 import kaldi_io as kio
    from paper_1909_08723_b200.errors import FormatError
    path = tmp_path / "idx.scp"
    for blob, want, etype, msg in load_golden("scp_cases.pkl.gz"):
        path.write_bytes(blob)
        if want is not None:
            got = [(e.utt_id, e.ark_path, e.offset) for e in kio.read_scp(str(path))]
            assert got == want, blob
        else:
            assert etype == "FormatError"
            with pytest.raises(FormatError) as ei:
                kio.read_scp(str(path))
            assert str(ei.value).replace(str(path), "idx.scp") == msg, blob


def test_ark_append_bytes_match_reference_layout(tmp_path):
    """write_ark_matrix (native appender) then read back: offsets, SCP lines
    and the reader round trip; the record bytes follow kaldi_io.py:129-150."""
    import struct
    from paper_1909_08723_b200 import kaldi_io as kio
    ark, scp = str(tmp_path / "o.ark"), str(tmp_path / "o.scp")
    rng = np.random.default_rng(3)
    mats = [rng.standard_normal((r, 5)).astype(np.float32) for r in (3, 1, 7)]
    offs = [kio.write_ark_matrix(f"u{i}", m_, ark, scp) for i, m_ in enumerate(mats)]
    blob = open(ark, "rb").read()
    pos = 0
    for i, (m_, o) in enumerate(zip(mats, offs)):
        head = f"u{i} ".encode()
        assert blob[pos:pos + len(head)] == head and o == pos + len(head)
        rec = b"\x00BFM \x04" + struct.pack("<i", m_.shape[0]) + b"\x04" + \
            struct.pack("<i", m_.shape[1]) + m_.astype("<f4").tobytes()
        assert blob[o:o + len(rec)] == rec
        pos = o + len(rec)
    assert pos == len(blob)
    ents = kio.read_scp(scp)
    assert [(e.utt_id, e.ark_path, e.offset) for e in ents] == \
        [(f"u{i}", ark, o) for i, o in enumerate(offs)]
    for e, m_ in zip(ents, mats):
        np.testing.assert_array_equal(kio.read_feature(e).data, m_)
    for bad in ("", "a b"):
        with pytest.raises(ValueError):
            kio.write_ark_matrix(bad, mats[0], ark, scp)
    with pytest.raises(ValueError):
        kio.write_ark_matrix("x", np.zeros((0, 3), np.float32), ark, scp)
    with pytest.raises(ValueError):
        kio.write_ark_matrix("x", np.full((1, 2), np.nan, np.float32), ark, scp)

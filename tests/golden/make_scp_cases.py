"""SCP parsing cases recorded from the UNMODIFIED reference ``read_scp``
(kaldi_io.py:46-77), run in the build container:

    python tests/golden/make_scp_cases.py

Each case is the file's bytes and either the parsed entries or the exception
type and message (the path inside messages is the placeholder file name
``idx.scp``).  ``tests/test_formats.py`` replays them through the native
parser.  Covers CRLF / lone CR line ends, unicode whitespace, blank lines,
int() spellings (sign, underscores, padding), paths containing ':' and
spaces, and every error kind.
"""

from __future__ import annotations

import gzip
import os
import pickle
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from fusedbeam.kaldi_io import read_scp  # noqa: E402

CASES = [
    b"a x.ark:5\nb y.ark:10\n",
    b"a x.ark:5\r\nb y.ark:10\r\n",
    b"a x.ark:5\rb y.ark:10\r",
    b"\n\n  a   x.ark:5  \n\t\nb\ty.ark:7",
    b"a c:/dir/x.ark:12\n",
    b"a dir with space/x.ark:3\n",
    b"a x.ark: 5\n",
    b"a x.ark:+5\n",
    b"a x.ark:1_000\n",
    b"a x.ark:00012\n",
    "a\u3000x.ark:4\nb\u00a0y.ark:6\n".encode(),
    "a x.ark:4\u2003\n".encode(),
    "\u00e9t\u00e9 x.ark:9\n".encode(),
    b"onlyone\n",
    b"a x.ark\n",
    b"a :5\n",
    b"a x.ark:five\n",
    b"a x.ark:1__0\n",
    b"a x.ark:_10\n",
    b"a x.ark:10_\n",
    b"a x.ark:\n",
    b"a x.ark:-3\n",
    b"a x.ark:5\nb y.ark:6\na z.ark:7\n",
    b"a x.ark:5\r\n\r\nb y.ark:6\r\na z.ark:7\r\n",
    b"a x.ark:'q'\n",
    b"",
    b"   \n\n",
]


def main():
    out = []
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "idx.scp")
        for blob in CASES:
            with open(path, "wb") as f:
                f.write(blob)
            try:
                res = [(e.utt_id, e.ark_path, e.offset) for e in read_scp(path)]
                out.append((blob, res, None, None))
            except Exception as e:      # noqa: BLE001
                out.append((blob, None, type(e).__name__, str(e).replace(path, "idx.scp")))
    with gzip.open(os.path.join(HERE, "scp_cases.pkl.gz"), "wb") as f:
        pickle.dump(out, f, protocol=4)
    for b, r, t, m in out:
        print(b[:40], r if r is not None else (t, m))


if __name__ == "__main__":
    main()

"""Kaldi SCP/ARK ingestion (reference ``kaldi_io.py``), natively read.

* ``FeatureMatrix`` / ``ScpEntry`` -- the reference records (``kaldi_io.py:31-41``).
* ``read_scp`` -- SCP index parsing (native ``fb_scp_parse``) with the
  reference's errors (``:46-77``).
* ``read_ark_matrix`` / ``read_feature`` -- one binary float32 record
  (``:82-134``), parsed by the C++ reader ``fb_ark_read_matrix``.
* ``write_ark_matrix`` -- append a record + SCP line (native
  ``fb_ark_append_matrix``; reference ``:129-150``).
* ``read_features_pinned`` -- a whole batch read by the C++ thread pool
  (``fb_ark_read_batch``) into ONE pinned host buffer: the FeatureMatrix data
  are views into it, so ``decode_batch``'s host->device copy starts from pinned
  memory.  Errors are the reference's (FormatError / IOError).
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import List, Sequence

import numpy as np

from . import _lib
from .errors import FormatError

BINARY_MARKER = b"\x00B"
FLOAT_MATRIX_TOKEN = b"FM "


@dataclass(frozen=True)
class ScpEntry:
    utt_id: str
    ark_path: str
    offset: int


@dataclass
class FeatureMatrix:
    utt_id: str
    data: np.ndarray   # [T, D] float32


def read_scp(path: str) -> List[ScpEntry]:
    """``utt_id path:offset`` lines, in order (reference kaldi_io.py:46-77),
    parsed natively (``fb_scp_parse``); the error texts are the reference's."""
    with open(path, "rb") as f:
        blob = f.read()
    blob.decode("utf-8")            # the reference reads text: same decode errors
    n_max = blob.count(b"\n") + blob.count(b"\r") + 1
    out = C.create_string_buffer(len(blob) + 2 * n_max + 16)
    offs = np.zeros(n_max, np.int64)
    out_len, n, err = C.c_int64(), C.c_int32(), (C.c_int32 * 3)()
    rc = _lib.lib().fb_scp_parse(blob, len(blob), out, len(out), C.byref(out_len),
                                 offs.ctypes.data, C.byref(n), err)
    if rc == 4:                     # FB_ERR_FORMAT: kind, line, first line; text in out
        kind, line, first = err[0], err[1], err[2]
        text = out.raw[:out_len.value].decode("utf-8")
        where = f"{path}:{line}"
        if kind == 1:
            raise FormatError(f"{where}: expected 'utt_id path:offset'")
        if kind == 2:
            raise FormatError(f"{where}: missing ':offset' suffix")
        if kind == 3:
            raise FormatError(f"{where}: offset {text!r} is not an integer")
        if kind == 4:
            raise FormatError(f"{where}: negative offset {int(text)}")
        raise FormatError(f"{where}: duplicate utterance id {text!r} (first seen on line {first})")
    _lib.check(rc)
    fields = out.raw[:out_len.value].split(b"\0")
    return [ScpEntry(fields[2 * i].decode("utf-8"), fields[2 * i + 1].decode("utf-8"),
                     int(offs[i])) for i in range(n.value)]


def _dims(ark_path: str, offset: int):
    r, c = C.c_int32(), C.c_int32()
    _lib.call("fb_ark_read_matrix", ark_path.encode(), offset, None, 0, C.byref(r), C.byref(c))
    return r.value, c.value


def read_ark_matrix(ark_path: str, offset: int) -> np.ndarray:
    """The float32 matrix at ``offset`` (reference kaldi_io.py:82-130)."""
    rows, cols = _dims(ark_path, offset)
    out = np.empty((rows, cols), np.float32)
    r, c = C.c_int32(), C.c_int32()
    _lib.call("fb_ark_read_matrix", ark_path.encode(), offset, out.ctypes.data, out.size,
              C.byref(r), C.byref(c))
    return out


def read_feature(entry: ScpEntry) -> FeatureMatrix:
    return FeatureMatrix(entry.utt_id, read_ark_matrix(entry.ark_path, entry.offset))


def read_features_pinned(entries: Sequence[ScpEntry], threads: int = 8) -> List[FeatureMatrix]:
    """Batch read into one pinned host buffer (C++ thread pool)."""
    import torch
    n = len(entries)
    if n == 0:
        return []
    paths = [e.ark_path.encode() for e in entries]
    c_paths = (C.c_char_p * n)(*paths)
    offs = np.asarray([e.offset for e in entries], np.int64)
    rows = np.zeros(n, np.int32)
    cols = np.zeros(n, np.int32)
    _lib.call("fb_ark_read_batch", n, C.cast(c_paths, C.c_void_p), offs.ctypes.data, None, None,
              None, rows.ctypes.data, cols.ctypes.data, threads)
    sizes = rows.astype(np.int64) * cols
    dst_off = np.zeros(n, np.int64)
    np.cumsum(sizes[:-1], out=dst_off[1:])
    buf = torch.empty(int(sizes.sum()), dtype=torch.float32,
                      pin_memory=torch.cuda.is_available())
    _lib.call("fb_ark_read_batch", n, C.cast(c_paths, C.c_void_p), offs.ctypes.data,
              buf.data_ptr(), dst_off.ctypes.data, sizes.ctypes.data, rows.ctypes.data,
              cols.ctypes.data, threads)
    host = buf.numpy()
    return [FeatureMatrix(e.utt_id, host[o:o + s].reshape(r, c))
            for e, o, s, r, c in zip(entries, dst_off, sizes, rows, cols)]


def write_ark_matrix(utt_id: str, matrix: np.ndarray, ark_path: str, scp_path: str) -> int:
    """Append one binary record and its SCP line (reference kaldi_io.py:129-150);
    returns the record's offset.  Same ValueErrors; the bytes are written by
    the native appender (``fb_ark_append_matrix``)."""
    if not utt_id or any(ch.isspace() for ch in utt_id):
        raise ValueError(f"bad utterance id {utt_id!r}")
    mat = np.ascontiguousarray(matrix, dtype="<f4")
    if mat.ndim != 2 or mat.shape[0] < 1 or mat.shape[1] < 1:
        raise ValueError(f"matrix must be 2-D and non-empty, got shape {mat.shape}")
    if not np.isfinite(mat).all():
        raise ValueError("matrix contains non-finite values")
    off = C.c_int64()
    _lib.call("fb_ark_append_matrix", os.fsencode(ark_path), os.fsencode(scp_path),
              utt_id.encode("utf-8"), mat.ctypes.data, mat.shape[0], mat.shape[1], C.byref(off))
    return off.value

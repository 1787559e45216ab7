"""Kaldi SCP/ARK ingestion (reference ``kaldi_io.py``), natively read.

* ``FeatureMatrix`` / ``ScpEntry`` -- the reference records (``kaldi_io.py:31-41``).
* ``read_scp`` -- SCP index parsing with the reference's errors (``:44-79``).
* ``read_ark_matrix`` / ``read_feature`` -- one binary float32 record
  (``:82-134``), parsed by the C++ reader ``fb_ark_read_matrix``.
* ``write_ark_matrix`` -- append a record + SCP line (``:137-160``).
* ``read_features_pinned`` -- a whole batch read by the C++ thread pool
  (``fb_ark_read_batch``) into ONE pinned host buffer: the FeatureMatrix data
  are views into it, so ``decode_batch``'s host->device copy starts from pinned
  memory.  Errors are the reference's (FormatError / IOError).
"""

from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass
from typing import List, Sequence

import numpy as np

from . import _lib
from .errors import FormatError

BINARY_MARKER = b"\x00B"
FLOAT_MATRIX_TOKEN = b"FM "
_INT_SIZE = b"\x04"


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
    """``utt_id path:offset`` lines, in order (reference kaldi_io.py:44-79)."""
    entries: List[ScpEntry] = []
    seen = {}
    with open(path, "r", encoding="utf-8") as f:
        for lineno, raw in enumerate(f, start=1):
            line = raw.strip()
            if not line:
                continue
            fields = line.split(None, 1)
            if len(fields) != 2:
                raise FormatError(f"{path}:{lineno}: expected 'utt_id path:offset'")
            utt_id, rest = fields
            ark_path, sep, offset_text = rest.rpartition(":")
            if not sep or not ark_path:
                raise FormatError(f"{path}:{lineno}: missing ':offset' suffix")
            try:
                offset = int(offset_text)
            except ValueError:
                raise FormatError(
                    f"{path}:{lineno}: offset {offset_text!r} is not an integer") from None
            if offset < 0:
                raise FormatError(f"{path}:{lineno}: negative offset {offset}")
            if utt_id in seen:
                raise FormatError(f"{path}:{lineno}: duplicate utterance id {utt_id!r}"
                                  f" (first seen on line {seen[utt_id]})")
            seen[utt_id] = lineno
            entries.append(ScpEntry(utt_id, ark_path, offset))
    return entries


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
    """Append one record + its SCP line; returns the offset (kaldi_io.py:137-160)."""
    if not utt_id or any(c.isspace() for c in utt_id):
        raise ValueError(f"bad utterance id {utt_id!r}")
    data = np.asarray(matrix, dtype=np.float32)
    if data.ndim != 2 or data.shape[0] < 1 or data.shape[1] < 1:
        raise ValueError(f"matrix must be 2-D and non-empty, got shape {data.shape}")
    if not np.isfinite(data).all():
        raise ValueError("matrix contains non-finite values")
    rows, cols = data.shape
    with open(ark_path, "ab") as ark:
        ark.write(utt_id.encode("utf-8") + b" ")
        offset = ark.tell()
        ark.write(BINARY_MARKER)
        ark.write(FLOAT_MATRIX_TOKEN)
        ark.write(_INT_SIZE + struct.pack("<i", rows))
        ark.write(_INT_SIZE + struct.pack("<i", cols))
        ark.write(np.ascontiguousarray(data, dtype="<f4").tobytes())
    with open(scp_path, "a", encoding="utf-8") as scp:
        scp.write(f"{utt_id} {ark_path}:{offset}\n")
    return offset

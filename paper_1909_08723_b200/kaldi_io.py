"""Feature container of the decoder API (reference ``kaldi_io.py:37-41``).

Kaldi SCP/ARK ingestion itself is out of scope for the device path (SURVEY.md
§2 row 11, §8f rank 3); only the record type ``decode_batch`` consumes lives here.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class FeatureMatrix:
    utt_id: str
    data: np.ndarray   # [T, D] float32

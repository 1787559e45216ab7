"""Shared pytest setup: the ``gpu`` marker, repo on sys.path, golden loaders."""

from __future__ import annotations

import gzip
import os
import pickle
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")


def load_golden(name: str):
    with gzip.open(os.path.join(GOLDEN, name), "rb") as f:
        return pickle.load(f)


@pytest.fixture(scope="session")
def cuda_lib():
    """The in-tree C-ABI library on a GPU box; fails loudly when it is missing."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1909_08723_b200 import _lib
    return _lib.lib()

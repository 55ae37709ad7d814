"""Shared fixtures.  Markers: ``gpu`` = needs a B200 (run with -m gpu)."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); the product path has no CPU fallback")
    config.addinivalue_line("markers", "slow: long-running full-size parity case")


@pytest.fixture(scope="session")
def cuda():
    """GPU tests fail (not skip) when the device or the extension is absent:
    a silent skip on the GPU box would hide a missing native path."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    from paper_2002_05018_b200 import _lib
    _lib.load()
    return torch


@pytest.fixture(scope="session")
def oracle():
    from oracle import d3m_oracle
    d3m_oracle.lib()
    return d3m_oracle


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def rand_complex_symmetric(n, seed, scale=1.0):
    """pkg/tests/conftest.py:11-14 generator."""
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    return scale * (G + G.T) / 2.0


def permuted(M, perm):
    return M[np.ix_(perm, perm)]


def reconstruct(fac):
    return fac.L @ fac.dense_d() @ fac.L.T


def split_blocks(x, sizes):
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(int)
    return [x[off[i]:off[i + 1]] for i in range(len(sizes))]


def reference_available() -> bool:
    return os.path.isdir(REFERENCE_SRC)

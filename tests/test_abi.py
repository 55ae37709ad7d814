"""CPU-side checks of the boundary: the C-ABI library loads, exports every
symbol include/d3m.h declares, and the Python binding covers them.  No
compute calls (no GPU here)."""

from __future__ import annotations

import ctypes
import os
import re

from conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "d3m.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|size_t|void\*?|const char\*)\s+(d3m_\w+)\s*\(", src, re.M)))


def test_header_declares_entry_points():
    names = _declared()
    for must in ("d3m_bk_factor_batched", "d3m_ldlt_solve_batched", "d3m_schur_reduce_batched",
                 "d3m_block_ldlt_exec", "d3m_block_solve_exec", "d3m_recover_batched", "d3m_zgemm_grouped"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2002_05018_b200 import build_ext
    path = build_ext.build()
    lib = ctypes.CDLL(path)
    for name in _declared():
        assert hasattr(lib, name), name
    from paper_2002_05018_b200 import _lib
    assert set(_declared()) <= set(_lib.exported_symbols())
    assert lib.d3m_abi_version() == _lib.ABI_VERSION == 13


def test_gpu_path_fails_loudly_without_device():
    import torch
    if torch.cuda.is_available():
        return
    import numpy as np
    import pytest
    from paper_2002_05018_b200 import D3MUnavailable, dense_ldlt_bk
    with pytest.raises(D3MUnavailable):
        dense_ldlt_bk(np.eye(3, dtype=complex))


def test_flow_extra_counters_match_header():
    import re
    from paper_2002_05018_b200 import _lib
    hdr = open(os.path.join(ROOT, "include", "d3m.h")).read()
    assert int(re.search(r"#define D3M_FLOW_EXTRA_COUNTERS (\d+)", hdr).group(1)) == _lib.FLOW_EXTRA_COUNTERS

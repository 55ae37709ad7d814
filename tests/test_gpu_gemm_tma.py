"""GPU parity: the TMA-staged update GEMM (zgemm3m_tma_kernel) against the
cp.async half-tile kernel on the same panel tasks -- bitwise -- and against
numpy (factor.py:213-230 trailing updates)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import rand_complex_symmetric

pytestmark = pytest.mark.gpu


def _tasks(_lib, n, blocks_x, blocks_l, pairs, ldcs, c_offs, sym_flags):
    t = np.zeros(len(pairs), dtype=_lib.GEMM_TASK)
    xo = np.concatenate([[0], np.cumsum(blocks_x)])
    lo = np.concatenate([[0], np.cumsum(blocks_l)])
    for q, (a, b) in enumerate(pairs):
        t[q]["a_off"] = xo[a] * n
        t[q]["b_off"] = lo[b] * n
        t[q]["c_off"] = c_offs[q]
        t[q]["m"], t[q]["n"], t[q]["k"] = blocks_x[a], blocks_l[b], n
        t[q]["lda"] = t[q]["ldb"] = n
        t[q]["ldc"] = ldcs[q]
        t[q]["flags"] = _lib.GEMM_SUB | (_lib.GEMM_SYM if sym_flags[q] else 0)
    return t


@pytest.mark.parametrize("n", [256, 200, 447, 24, 9])
def test_tma_update_is_bitwise_the_half_tile_kernel(cuda, n):
    from paper_2002_05018_b200 import _lib
    from paper_2002_05018_b200.device import stream_ptr, to_device
    rng = np.random.default_rng(100 + n)
    blocks = [n, 130, 64, 257 if n > 64 else 70]           # block rows of the panel (ragged tiles)
    R = sum(blocks)
    X = rng.standard_normal((R, n)) + 1j * rng.standard_normal((R, n))
    L = rng.standard_normal((R, n)) + 1j * rng.standard_normal((R, n))
    # targets: every pair (a >= b); diagonal pairs are symmetric targets
    pairs = [(a, b) for a in range(len(blocks)) for b in range(a + 1)]
    sizes = [blocks[a] * blocks[b] for a, b in pairs]
    c_offs = np.concatenate([[0], np.cumsum(sizes)])[:-1]
    ldcs = [blocks[b] for _, b in pairs]
    symf = [a == b for a, b in pairs]
    C0 = rng.standard_normal(sum(sizes)) + 1j * rng.standard_normal(sum(sizes))
    for q, (a, b) in enumerate(pairs):                     # symmetric targets start symmetric
        if a == b:
            m = blocks[a]
            C0[c_offs[q]:c_offs[q] + m * m] = rand_complex_symmetric(m, q).ravel()
    dX, dL = to_device(X), to_device(L)
    dt = cuda.empty(64 * len(pairs), dtype=cuda.uint8, device="cuda")
    # reference: the cp.async kernel
    t = _tasks(_lib, n, blocks, blocks, pairs, ldcs, c_offs, symf)
    dC1 = to_device(C0.copy())
    _lib.call("d3m_zgemm_grouped", 0, 0, _lib.ptr(dX), _lib.ptr(dL), _lib.ptr(dC1), _lib.hptr(t), len(t),
              _lib.ptr(dt), stream_ptr())
    want = dC1.cpu().numpy()
    t = _tasks(_lib, n, blocks, blocks, pairs, ldcs, c_offs, symf)
    dC2 = to_device(C0.copy())
    _lib.call("d3m_zgemm_tma_panels", _lib.ptr(dX), R, _lib.ptr(dL), R, n, _lib.ptr(dC2), _lib.hptr(t), len(t),
              _lib.ptr(dt), stream_ptr())
    got = dC2.cpu().numpy()
    assert np.array_equal(got, want)
    # and against numpy on one off-diagonal and one diagonal target
    xo = np.concatenate([[0], np.cumsum(blocks)])
    for q, (a, b) in enumerate(pairs):
        if (a, b) not in ((2, 1), (3, 3)):
            continue
        upd = X[xo[a]:xo[a + 1]] @ L[xo[b]:xo[b + 1]].T
        ref = C0[c_offs[q]:c_offs[q] + sizes[q]].reshape(blocks[a], blocks[b])
        if a == b:
            upd = np.tril(upd) + np.tril(upd, -1).T
        blk = got[c_offs[q]:c_offs[q] + sizes[q]].reshape(blocks[a], blocks[b])
        assert np.abs(blk - (ref - upd)).max() <= 1e-12 * max(1.0, np.abs(upd).max())


def test_tma_rejects_tasks_outside_the_panel_form(cuda):
    from paper_2002_05018_b200 import _lib
    from paper_2002_05018_b200.device import stream_ptr, to_device
    X = to_device(np.ones((64, 32), complex))
    C = to_device(np.zeros((64, 64), complex))
    t = np.zeros(1, dtype=_lib.GEMM_TASK)
    t["m"], t["n"], t["k"], t["lda"], t["ldb"], t["ldc"] = 64, 64, 32, 40, 32, 64      # lda != n
    dt = cuda.empty(64, dtype=cuda.uint8, device="cuda")
    with pytest.raises(_lib.D3MError):
        _lib.call("d3m_zgemm_tma_panels", _lib.ptr(X), 64, _lib.ptr(X), 64, 32, _lib.ptr(C), _lib.hptr(t), 1,
                  _lib.ptr(dt), stream_ptr())

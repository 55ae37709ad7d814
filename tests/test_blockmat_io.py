"""The "D3M-BLK v1" golden-K exchange format (blockmat.py:132-177): our
save_blk writes the reference's dump byte for byte, load_blk reads the
reference's own dump (tests/golden/k_small.blk, written by the reference's
save_blk in tools/gen_golden.py gen_blk) into bit-identical blocks, round
trips are exact, and malformed files raise the reference's errors.  The GPU
test factors the loaded dump against the reference's pivots and solution."""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import ROOT, golden

BLK = os.path.join(ROOT, "tests", "golden", "k_small.blk")


def test_load_reference_dump_and_rewrite_byte_identical(tmp_path):
    from paper_2002_05018_b200 import blockmat as bm
    from paper_2002_05018_b200 import workloads as wl
    K = bm.load_blk(BLK)
    Kw = wl.config4_matrix(seed=21, grid=(2, 2, 3), n=12)          # the generator the dump was made from
    assert list(K.sizes) == list(Kw.sizes) and set(K.blocks) == set(Kw.blocks)
    for k, b in Kw.blocks.items():
        assert np.array_equal(np.asarray(K.blocks[k]), np.asarray(b)), k
    out = tmp_path / "k.blk"
    bm.save_blk(out, K)
    assert out.read_bytes() == open(BLK, "rb").read()


def test_round_trip_edge_cases(tmp_path):
    from paper_2002_05018_b200 import blockmat as bm
    rng = np.random.default_rng(3)
    sizes = [1, 3, 0, 2]
    z = (rng.standard_normal((3, 3)) + 1j * rng.standard_normal((3, 3)))
    trip = [(0, 0, np.array([[1e-300 - 2.5e300j]])), (1, 1, z + z.T), (3, 1, rng.standard_normal((2, 3)) + 0j),
            (3, 3, np.array([[np.pi, 1j], [1j, -0.0]]))]
    K = bm.from_blocks(sizes, trip)
    p = tmp_path / "e.blk"
    bm.save_blk(p, K)
    K2 = bm.load_blk(p)
    for k, b in K.blocks.items():
        assert np.array_equal(np.asarray(K2.blocks[k]), np.asarray(b))
        assert np.array_equal(np.signbit(np.asarray(K2.blocks[k]).real), np.signbit(np.asarray(b).real))


@pytest.mark.parametrize("text,msg", [
    ("D3M-BLK v0\n1 1\n0 0\n1 0\n", "bad magic line"),
    ("D3M-BLK v1\n", "missing header line"),
    ("D3M-BLK v1\n2 1\n", "header size list does not match block count"),
    ("D3M-BLK v1\n1 2\n0 0\n1 0 2 0\n", "truncated data for block \\(0, 0\\)"),
])
def test_malformed_dumps_raise_reference_errors(tmp_path, text, msg):
    from paper_2002_05018_b200 import blockmat as bm
    p = tmp_path / "bad.blk"
    p.write_text(text)
    with pytest.raises(bm.BlockMatrixError, match=msg):
        bm.load_blk(p)


@pytest.mark.gpu
def test_factor_reference_dump_vs_reference(cuda):
    """K loaded from the reference's dump factors with the reference's
    ordering and pivots bit-exactly; the solution agrees to 1e-9."""
    import paper_2002_05018_b200 as d
    g = golden("k_small.npz")
    K = d.load_blk(BLK)
    gr = d.clique_graph(K)
    order = d.reorder(gr, K.sizes)
    assert np.array_equal(order.perm, g["order"])
    F = d.block_ldlt(K, d.symbolic_factor(gr, order, K.sizes))
    assert np.array_equal(np.concatenate([f.perm for f in F.diag]), g["perm"])
    assert np.array_equal(np.concatenate([f.tags for f in F.diag]), g["tags"])
    off = np.concatenate([[0], np.cumsum(K.sizes)])
    b = [g["b"][off[i]:off[i + 1]] for i in range(K.nblocks)]
    x = np.concatenate([np.asarray(v) for v in d.block_solve(F, b)])
    assert np.linalg.norm(x - g["x"]) <= 1e-9 * np.linalg.norm(g["x"])

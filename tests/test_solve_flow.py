"""Host checks of the native planner (csrc/d3m_plan.cpp, no GPU needed).

The dataflow block-solve work list (factor.flow_items): every item's
dependencies are satisfied by the items before it (so the device queue,
which hands items out in list order, cannot deadlock), each 16-row tile
receives its updates in ascending column order, every counter reaches the
value the later items wait for, and the list equals the pure-Python
restatement (tests/ref/flow_ref.py).  The block_ldlt GEMM task table equals
its Python restatement (tests/ref/schedule_ref.py) record for record."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2002_05018_b200 import planner, workloads as wl
from paper_2002_05018_b200.blockmat import clique_graph
from paper_2002_05018_b200.factor import _BC, _BE, _BR, _FA, _FB, _FD, flow_items
from paper_2002_05018_b200.ordering import identity_ordering, reorder
from paper_2002_05018_b200.symbolic import symbolic_factor


def _check(plan):
    sizes = np.asarray(plan.sizes_perm, dtype=np.int64)
    pattern = [np.asarray(p, dtype=np.int64) for p in plan.pattern]
    panel_rows = np.array([int(sizes[p].sum()) for p in pattern], dtype=np.int64)
    items, deps, part_off, ncnt, part_elems = flow_items(sizes, pattern, panel_rows)
    from ref.flow_ref import flow_items_ref
    ref = flow_items_ref(sizes, pattern, panel_rows)
    assert np.array_equal(items, ref[0]) and np.array_equal(deps, ref[1]) and np.array_equal(part_off, ref[2])
    assert (ncnt, part_elems) == ref[3:]
    _check_tasks(sizes, pattern)
    cnt = np.zeros(ncnt, dtype=np.int64)
    upd_order = {}
    for idx, (typ, j, p0, p1, doff, dcnt, inc0, inc1) in enumerate(items):
        for c, target in deps[doff:doff + dcnt]:
            assert cnt[c] >= target, (idx, typ, j, c, target, cnt[c])
        if typ == _FB:
            upd_order.setdefault((j, p0), None)
        for c in (inc0, inc1):
            if c >= 0:
                cnt[c] += 1
    nb = len(sizes)
    T = (sizes + 15) // 16
    assert np.array_equal(cnt[:nb], np.where(sizes > 0, T, 0))                   # z tiles
    assert np.array_equal(cnt[5 * nb:6 * nb], np.where(sizes > 0, T, 0))         # x tiles
    # every update tile of every column appears exactly once
    fb = items[items[:, 0] == _FB]
    expect = sum(int(T[i]) for j in range(nb) for i in pattern[j])
    assert len(fb) == expect
    # per target tile: ascending columns
    seen = {}
    for typ, j, p0, p1, *_ in items:
        if typ != _FB:
            continue
        tgt = (int(np.searchsorted(np.cumsum(sizes[pattern[j]]), p0, side="right")), j)
        i = int(pattern[j][tgt[0]])
        t = (p0 - int(np.concatenate([[0], np.cumsum(sizes[pattern[j]])])[tgt[0]])) // 16
        last = seen.get((i, t), -1)
        assert j > last
        seen[(i, t)] = j
    assert part_elems >= 1 and len(part_off) >= 1
    return items


def _check_tasks(sizes, pattern):
    from ref.schedule_ref import gemm_tasks_ref
    nb = len(sizes)
    diag_off = np.zeros(nb, dtype=np.int64)
    panel_off = np.zeros(nb, dtype=np.int64)
    off = 0
    for j in range(nb):
        diag_off[j] = off
        off += int(sizes[j]) ** 2
        panel_off[j] = off
        off += int(sizes[pattern[j]].sum()) * int(sizes[j])
    got = planner.gemm_tasks(sizes, pattern, diag_off, panel_off)
    want = gemm_tasks_ref(sizes, pattern, diag_off, panel_off)
    assert got[0].tobytes() == want[0].tobytes()
    for a, b in zip(got[1:5], want[1:5]):
        assert np.array_equal(a, b)
    assert got[5] == want[5]


def test_gemm_tasks_reject_targets_outside_pattern():
    sizes = np.array([2, 3, 4], dtype=np.int64)
    pattern = [np.array([1, 2]), np.array([], dtype=np.int64), np.array([], dtype=np.int64)]   # (2, 1) missing
    with pytest.raises(ValueError, match="outside the pattern"):
        planner.gemm_tasks(sizes, pattern, np.zeros(3, np.int64), np.zeros(3, np.int64))


def test_flow_list_config4():
    """Config 4's plan (144 faces x 256, natural order): structure from the
    face adjacency with 1x1 placeholder blocks."""
    from paper_2002_05018_b200.blockmat import from_blocks
    from paper_2002_05018_b200.workloads import grid_faces
    faces = grid_faces(4, 4, 4)
    trip = [(f, g, np.ones((1, 1))) for f in range(len(faces)) for g in range(f + 1)
            if f == g or set(faces[f]) & set(faces[g])]
    K1 = from_blocks([1] * len(faces), trip)
    plan = symbolic_factor(clique_graph(K1), identity_ordering(len(faces)), [256] * len(faces))
    items = _check(plan)
    assert len(items) > 100_000


@pytest.mark.parametrize("seed", range(12))
def test_flow_list_random_plans(seed):
    K, _ = wl.rand_block_system(seed + 200, max_blocks=14, max_size=40, density=0.35)
    g = clique_graph(K)
    for order in (reorder(g, K.sizes), identity_ordering(K.nblocks)):
        _check(symbolic_factor(g, order, K.sizes))


def test_etree_schedule_dependencies():
    """planner.etree_schedule: a chain stays on one stream; in a forest the
    leaves of different subtrees take different streams; the recorded bulk
    writers are the last earlier columns whose pattern holds the column."""
    from paper_2002_05018_b200 import planner
    parent = np.array([1, 2, 3, -1])
    pattern = [np.array([1, 3]), np.array([2, 3]), np.array([3]), np.array([], dtype=np.int64)]
    s = planner.etree_schedule(parent, pattern).reshape(-1, 3)
    assert set(s[:, 0]) == {0}
    assert list(s[:, 1]) == [-1, -1, -1, 1]          # column 3: written by the rest updates of 0 and 1
    assert list(s[:, 2]) == [-1, -1, 1, -1]          # column 2 updates 3 after 1's rest update
    parent = np.array([2, 2, 5, 5, 5, -1])            # subtrees {0,1,2} and {3,4}
    pattern = [np.array([2, 5]), np.array([2]), np.array([5]), np.array([5]), np.array([5]),
               np.array([], dtype=np.int64)]
    s = planner.etree_schedule(parent, pattern).reshape(-1, 3)
    assert s[0, 0] != s[1, 0] and s[2, 0] == s[1, 0] and s[3, 0] != s[2, 0]
    assert s[5, 1] == 3                               # 4 -> 5 is a next update; 3 is the last rest writer


def test_chain_split_keeps_order_and_picks_the_critical_items():
    from paper_2002_05018_b200.factor import chain_split
    sizes = np.array([256, 200, 256, 130, 256, 64], dtype=np.int64)
    pattern = [np.array([1, 2, 4]), np.array([2, 5]), np.array([3, 4, 5]), np.array([4]), np.array([5]), np.array([])]
    panel_rows = np.array([int(sizes[p].sum()) if len(p) else 0 for p in pattern], dtype=np.int64)
    items = flow_items(sizes, pattern, panel_rows)[0]
    split, nchain = chain_split(items, sizes, pattern)
    assert len(split) == len(items) and 0 < nchain < len(items)
    key = {tuple(r): i for i, r in enumerate(items)}
    pos = np.array([key[tuple(r)] for r in split])
    assert np.all(np.diff(pos[:nchain]) > 0) and np.all(np.diff(pos[nchain:]) > 0)    # stable parts
    for r in split[:nchain]:
        typ, j, p0 = int(r[0]), int(r[1]), int(r[2])
        npar = int(sizes[pattern[j][0]]) if len(pattern[j]) else 0
        assert typ in (_FA, _BR, _BE) or (typ == _FB and p0 < npar) or (typ == _BC and 256 * p0 < npar)
    assert not np.any(split[nchain:, 0] == _FA) and np.all(split[:nchain, 0] != _FD)

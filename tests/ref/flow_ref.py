"""Pure-Python restatement of the dataflow solve's work list: the checker of
the C++ planner (paper_2002_05018_b200/csrc/d3m_plan.cpp d3m_plan_flow_items),
which must produce the identical list.  Test infrastructure only."""

from __future__ import annotations

import numpy as np

_FA, _FB, _FD, _BC, _BR, _BE = 0, 2, 1, 3, 4, 5      # skinny_dmma.cu FlowItem types
_KCH = 256
_FD_ROWS, _BR_ROWS = 32, 16


def flow_items_ref(sizes, pattern, panel_rows):
    """Host part of _solve_flow (pure numpy; tests/test_solve_flow.py checks
    that the list is a topological order).  Returns (items int32 [n, 8],
    deps int32 [m, 2], part_off int64 [nb], counter count, partial elems)."""
    nb = len(sizes)
    sizes = [int(v) for v in sizes]
    T = [(n + 15) // 16 for n in sizes]
    pat = [[int(i) for i in p] for p in pattern]
    prow = [dict() for _ in range(nb)]                 # panel row offset of target block i in panel j
    for j in range(nb):
        r = 0
        for i in pat[j]:
            prow[j][i] = r
            r += sizes[i]
    ZC, BLK, UC, CC, RC, XC = (k * nb for k in range(6))
    seq_base = np.concatenate([[6 * nb], 6 * nb + np.cumsum(T)]).astype(np.int64)
    ncnt = int(seq_base[-1]) + 1                       # + queue head
    items, deps = [], []

    def add(typ, j, p0, p1, dl, inc0, inc1=-1):
        items.append((typ, j, p0, p1, len(deps), len(dl), inc0, inc1))
        deps.extend(dl)

    n_into = [0] * nb                                  # FB tile items into each block
    for j in range(nb):
        for i in pat[j]:
            n_into[i] += T[i]
    seq_k = [[0] * T[i] for i in range(nb)]

    def update(j, i):
        for t in range(T[i]):
            rows = min(16, sizes[i] - 16 * t)
            add(_FB, j, prow[j][i] + 16 * t, rows, [(ZC + j, T[j]), (int(seq_base[i]) + t, seq_k[i][t])],
                int(seq_base[i]) + t, BLK + i)
            seq_k[i][t] += 1

    pending = [[] for _ in range(nb)]                  # deferred updates (column j) per target block, FIFO

    def flush(i, upto=None):
        while pending[i] and (upto is None or pending[i][0] <= upto):
            update(pending[i].pop(0), i)

    for j in range(nb):
        if sizes[j]:
            for t in range(T[j]):
                add(_FA, j, t, 0, [(BLK + j, n_into[j])] if n_into[j] else [], ZC + j)
            for r0 in range(0, sizes[j], _FD_ROWS):
                add(_FD, j, r0, min(sizes[j], r0 + _FD_ROWS), [(ZC + j, T[j])], UC + j)
        if pat[j]:
            par = pat[j][0]
            flush(par)
            update(j, par)
        if j >= 1:
            for i in pat[j - 1][1:]:
                flush(i, upto=j - 1)
        for i in pat[j][1:]:
            pending[i].append(j)
    for i in range(nb):
        flush(i)
    # backward
    nch = [(int(panel_rows[j]) + _KCH - 1) // _KCH for j in range(nb)]

    def chunk_blocks(j, ch):
        lo, hi = ch * _KCH, min(int(panel_rows[j]), ch * _KCH + _KCH)
        return [i for i in pat[j] if prow[j][i] < hi and prow[j][i] + sizes[i] > lo and sizes[i]]

    def parent_chunk(j, ch):
        return bool(pat[j]) and pat[j][0] in chunk_blocks(j, ch)

    done_far = [False] * nb

    def chunks(j, far):
        for ch in range(nch[j]):
            if parent_chunk(j, ch) != far:
                for mt in range(T[j]):
                    add(_BC, j, ch, mt, [(XC + i, T[i]) for i in chunk_blocks(j, ch)], CC + j)

    for j in range(nb - 1, -1, -1):
        if not sizes[j]:
            continue
        if not done_far[j]:
            chunks(j, True)
            done_far[j] = True
        chunks(j, False)
        npc = (sizes[j] + _BR_ROWS - 1) // _BR_ROWS
        nfd = (sizes[j] + _FD_ROWS - 1) // _FD_ROWS
        for pc in range(npc):
            add(_BR, j, _BR_ROWS * pc, min(sizes[j], _BR_ROWS * pc + _BR_ROWS), [(CC + j, nch[j] * T[j]), (UC + j, nfd)],
                RC + j)
        for t in range(T[j]):
            add(_BE, j, t, 0, [(RC + j, npc)], XC + j)
        if j >= 1 and sizes[j - 1] and not done_far[j - 1]:
            chunks(j - 1, True)
            done_far[j - 1] = True
    part_off = np.zeros(max(nb, 1), dtype=np.int64)
    acc = 0
    for j in range(nb):
        part_off[j] = acc
        acc += nch[j] * sizes[j] * 16
    it = np.ascontiguousarray(np.asarray(items, dtype=np.int32).reshape(-1, 8))
    dp = np.ascontiguousarray(np.asarray(deps, dtype=np.int32).reshape(-1, 2) if deps else np.zeros((1, 2), np.int32))
    return it, dp, part_off, ncnt, max(acc, 1)

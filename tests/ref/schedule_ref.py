"""Pure-Python restatement of the block_ldlt trailing-update task table
(factor.py:209-219 as GEMM records): the checker of the native planner
(csrc/d3m_plan.cpp d3m_plan_gemm_tasks).  Test infrastructure only."""

from __future__ import annotations

import numpy as np

from paper_2002_05018_b200 import _lib


def gemm_tasks_ref(sizes, pattern, diag_off, panel_off):
    sizes = np.asarray(sizes, dtype=np.int64)
    nb = len(sizes)
    rowpos = {}
    for j in range(nb):
        r = 0
        for i in pattern[j]:
            rowpos[(int(i), j)] = r
            r += int(sizes[int(i)])
    recs, ptr, nxt, tiles_n, tiles_r = [], [0], [], [], []
    bm = _lib.GEMM_BM
    flops = 0
    for j in range(nb):
        nj = int(sizes[j])
        rows = [int(i) for i in pattern[j]]
        prow = np.concatenate([[0], np.cumsum(sizes[rows])]).astype(np.int64) if rows else [0]
        nxt_recs, rest_recs = [], []
        for a, i in enumerate(rows):
            for b in range(a + 1):
                kk = rows[b]
                ni, nk = int(sizes[i]), int(sizes[kk])
                if i == kk:
                    c_off, ldc, flags = int(diag_off[i]), ni, _lib.GEMM_SUB | _lib.GEMM_SYM
                    tm = (ni + bm - 1) // bm
                    tiles = tm * (tm + 1) // 2
                    flops += 4 * ni * ni * nj
                else:
                    if (i, kk) not in rowpos:
                        raise ValueError(f"update targets block {(i, kk)} outside pattern")
                    c_off, ldc, flags = int(panel_off[kk]) + rowpos[(i, kk)] * nk, nk, _lib.GEMM_SUB
                    tiles = ((ni + bm - 1) // bm) * ((nk + bm - 1) // bm)
                    flops += 8 * ni * nk * nj
                rec = (int(prow[a]) * nj, int(panel_off[j]) + int(prow[b]) * nj, c_off, ni, nk, nj,
                       nj, nj, ldc, flags, tiles, (nk + bm - 1) // bm)
                (nxt_recs if kk == j + 1 else rest_recs).append(rec)
        for group, tl in ((nxt_recs, tiles_n), (rest_recs, tiles_r)):
            start = 0
            for rec in group:
                recs.append(rec[:10] + (start, rec[11], 0))
                start += rec[10]
            tl.append(start)
        nxt.append(ptr[-1] + len(nxt_recs))
        ptr.append(ptr[-1] + len(nxt_recs) + len(rest_recs))
    tasks = np.zeros(len(recs), dtype=_lib.GEMM_TASK)
    if recs:
        arr = np.array(recs, dtype=np.int64)
        for c, name in enumerate(_lib.GEMM_TASK.names):
            tasks[name] = arr[:, c]
    return (tasks, np.asarray(ptr, dtype=np.int64), np.asarray(nxt or [0], dtype=np.int64),
            np.asarray(tiles_n or [0], dtype=np.int64), np.asarray(tiles_r or [0], dtype=np.int64), flops)

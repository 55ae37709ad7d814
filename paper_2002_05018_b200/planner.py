"""Host planning of the block factorisation and solve, in native code.

The tables depend only on the elimination plan (symbolic.py:36-64): the
trailing-update GEMM task table of block_ldlt (factor.py:209-219) and the
work list of the dataflow block solve (factor.py:243-310).  Both are built
by csrc/d3m_plan.cpp (host functions of libd3m; no device needed) in
milliseconds, where Python loops took about a second on a config-5-shaped
plan."""

from __future__ import annotations

import numpy as np

from . import _lib


def _pattern_csr(pattern):
    ptr = np.zeros(len(pattern) + 1, dtype=np.int64)
    ptr[1:] = np.cumsum([len(p) for p in pattern])
    idx = (np.concatenate([np.asarray(p, dtype=np.int64) for p in pattern]) if ptr[-1]
           else np.zeros(1, dtype=np.int64))
    return ptr, np.ascontiguousarray(idx, dtype=np.int64)


def gemm_tasks(sizes, pattern, diag_off, panel_off):
    """-> (tasks GEMM_TASK[n], task_ptr[nb+1], task_next[nb], tiles_next[nb],
    tiles_rest[nb], update flops).  Raises ValueError (caller maps it to
    FactorConsistencyError) when an update targets a block outside the
    pattern (factor.py:224-226)."""
    lib = _lib.load()
    nb = len(sizes)
    sizes = np.ascontiguousarray(sizes, dtype=np.int64)
    ptr, idx = _pattern_csr(pattern)
    diag_off = np.ascontiguousarray(diag_off, dtype=np.int64)
    panel_off = np.ascontiguousarray(panel_off, dtype=np.int64)
    H = _lib.hptr
    task_ptr = np.zeros(nb + 1, dtype=np.int64)
    task_next = np.zeros(max(nb, 1), dtype=np.int64)
    tiles_next = np.zeros(max(nb, 1), dtype=np.int64)
    tiles_rest = np.zeros(max(nb, 1), dtype=np.int64)
    flops = np.zeros(1, dtype=np.int64)
    null = _lib.ctypes.c_void_p(0)
    n = lib.d3m_plan_gemm_tasks(nb, H(sizes), H(ptr), H(idx), H(diag_off), H(panel_off), null, 0,
                                null, null, null, null, null)
    if n == -1:
        raise ValueError("update targets a block outside the pattern")
    tasks = np.zeros(max(n, 0), dtype=_lib.GEMM_TASK)
    rc = lib.d3m_plan_gemm_tasks(nb, H(sizes), H(ptr), H(idx), H(diag_off), H(panel_off),
                                 _lib.ctypes.c_void_p(tasks.ctypes.data) if n else null, n, H(task_ptr),
                                 H(task_next), H(tiles_next), H(tiles_rest), H(flops))
    if rc != n:
        raise RuntimeError(f"d3m_plan_gemm_tasks returned {rc}, expected {n}")
    return tasks, task_ptr, task_next, tiles_next, tiles_rest, int(flops[0])


def flow_items(sizes, pattern, panel_rows):
    """-> (items int32 [n, 8], deps int32 [m, 2] (>= 1 row), part_off int64
    [max(nb, 1)], counter count, partial-sum elements)."""
    lib = _lib.load()
    nb = len(sizes)
    sizes = np.ascontiguousarray(sizes, dtype=np.int64)
    ptr, idx = _pattern_csr(pattern)
    panel_rows = np.ascontiguousarray(panel_rows if nb else np.zeros(1), dtype=np.int64)
    H = _lib.hptr
    null = _lib.ctypes.c_void_p(0)
    out = np.zeros(4, dtype=np.int64)
    part_off = np.zeros(max(nb, 1), dtype=np.int64)
    rc = lib.d3m_plan_flow_items(nb, H(sizes), H(ptr), H(idx), H(panel_rows), null, 0, null, 0, null, H(out))
    if rc != 0:
        raise RuntimeError(f"d3m_plan_flow_items returned {rc}")
    ni, nd = int(out[0]), int(out[1])
    items = np.zeros((ni, 8), dtype=np.int32)
    deps = np.zeros((max(nd, 1), 2), dtype=np.int32)
    rc = lib.d3m_plan_flow_items(nb, H(sizes), H(ptr), H(idx), H(panel_rows), H(items), ni, H(deps), nd,
                                 H(part_off), H(out))
    if rc != 0:
        raise RuntimeError(f"d3m_plan_flow_items returned {rc}")
    return items, deps, part_off, int(out[2]), int(out[3])


N_CRIT_STREAMS = 4          # d3m_capi.cu kCritStreams


def etree_schedule(parent, pattern, nstreams: int = N_CRIT_STREAMS) -> np.ndarray:
    """Per block column j (plan order) the int32 triple the etree-parallel
    executor (include/d3m.h d3m_block_ldlt_exec, h_sched) needs:

    * the critical stream: the stream of j's last child, so a chain of the
      elimination tree stays on one stream; a leaf takes the stream whose
      last column is the oldest, so independent subtrees spread out;
    * the last column k < j whose bulk ("rest") update writes column j:
      max{k : j in pattern(k), j != k + 1} (-1: none; column k+1 is
      written by k's "next" update instead);
    * the last column k < j whose bulk update writes column j+1.
    """
    nb = len(pattern)
    out = np.full((max(nb, 1), 3), -1, dtype=np.int32)
    last_child = np.full(max(nb, 1), -1, dtype=np.int64)
    for j in range(nb):
        p = int(parent[j])
        if p >= 0:
            last_child[p] = max(last_child[p], j)
    last_use = np.full(nstreams, -1, dtype=np.int64)
    dep = np.full(nb + 1, -1, dtype=np.int64)          # last rest-writer seen so far, per target column
    for j in range(nb):
        c = int(last_child[j])
        q = int(out[c, 0]) if c >= 0 else int(np.argmin(last_use))
        out[j, 0] = q
        last_use[q] = j
        out[j, 1] = dep[j]
        out[j, 2] = dep[j + 1] if j + 1 <= nb else -1
        for t in pattern[j]:
            t = int(t)
            if t != j + 1:
                dep[t] = j
    if nb == 0:
        out[0] = (0, -1, -1)
    return np.ascontiguousarray(out.reshape(-1))

"""Numeric factorisation on the B200: dense Bunch-Kaufman LDL^T, the
right-looking block LDL^T over an elimination plan, block substitution.

Drop-in for the reference's factor.py (pkg/src/ddsolve/factor.py:1-334):
same names, signatures, dataclass fields, error types and messages.  All
numerics run in libd3m (sm_100a); this module plans device layouts, moves
data and raises the reference's exceptions from device pivot outcomes.

Device layout of a BlockFactor (one HBM pool, complex128):
  per block column j (plan order):  diagonal slot  n_j x n_j  (packed BK
  factor: strict lower = L_jj, diagonal = d, W[k+1,k] = e of 2x2 pivots)
  followed by the panel  R_j x n_j  stacking L_ij for i in pattern[j]
  (ascending), R_j = sum n_i.  Pivots: perm (int64) / tags (int8) at the
  plan-order row offset of the column.
"""

from __future__ import annotations

import threading
from collections import OrderedDict
from collections.abc import Mapping
from dataclasses import dataclass, field

import numpy as np

from . import _lib, planner
from .blockmat import BlockSparseSym
from .device import DeviceArray, empty, require_cuda, stream_ptr, to_device, upload_bytes, upload_i64
from .symbolic import EliminationPlan

DEFAULT_PIVOT_TOL = 1e-12      # factor.py:19
# block_solve kernel: "flow" (dataflow work items, default) or "barrier" (the
# grid-barrier persistent kernel / per-product launches, D3M_SOLVE=p|l)
import os as _os
_SOLVE_MODE = "barrier" if _os.environ.get("D3M_SOLVE", "")[:1] in ("p", "l") else "flow"
_P = _lib.ptr


class SingularBlockError(Exception):
    """Both 1x1 and 2x2 pivot candidates fell below the pivot threshold."""


class SolverStateError(Exception):
    """Factor state missing or released (subdomain.py:221-223 analog)."""


class FactorConsistencyError(Exception):
    """Numeric factorization touched a block outside the symbolic pattern."""


def _singular_msg(info: int, thr: float) -> str:
    return f"no acceptable pivot at elimination step {info} (threshold {thr:.3e})"     # factor.py:101-103


# ---------------------------------------------------------------------------
# Dense factor
# ---------------------------------------------------------------------------

class DenseFactor:
    """P M P^T = L D L^T with unit lower L and 1x1/2x2 block diagonal D.

    Device-resident: ``packed`` (n x n, kernels.py:7-22 storage), ``perm_dev``
    and ``tags_dev`` live in HBM; the reference's fields L, d, e, tags, perm
    are materialised on the host on first access.
    """

    def __init__(self, packed, perm_dev, tags_dev, growth: float, n_2x2: int):
        self.packed = packed            # torch (n, n) complex128 view (None once released)
        self.perm_dev = perm_dev        # torch (n,) int64 view
        self.tags_dev = tags_dev        # torch (n,) int8 view
        self.growth = float(growth)
        self.n_2x2 = int(n_2x2)
        self._n = int(perm_dev.shape[0])
        self._host = None
        # (decision margin, argmax gap) of the pivot sequence when the
        # factorisation tracked them (margins=True), else None: the minimum
        # relative distance of any BK test of kernels.py:59-77 to its
        # threshold and of the colmax winner to the runner-up
        self.margin = None

    @property
    def n(self) -> int:
        return self._n

    @property
    def released(self) -> bool:
        return self.packed is None

    def release(self) -> "DenseFactor":
        """Drop the factor values (keep perm / tags / stats); used by
        reduce_domains(keep="solution") when the factors do not fit in HBM."""
        self.packed = None
        return self

    def _unpack(self):
        if self._host is None:
            if self.packed is None:
                raise SolverStateError("factor values were released (reduce_domains keep='solution')")
            W = self.packed.cpu().numpy()
            tags = self.tags_dev.cpu().numpy().astype(np.int8)
            perm = self.perm_dev.cpu().numpy().astype(np.int64)
            n = W.shape[0]
            L = np.tril(W, -1)
            d = np.diagonal(W).copy()
            e = np.zeros(n, dtype=np.complex128)
            two = np.flatnonzero(tags == 2)
            e[two] = W[two + 1, two]
            L[two + 1, two] = 0.0
            np.fill_diagonal(L, 1.0)
            self._host = (L, d, e, tags, perm)
        return self._host

    L = property(lambda self: self._unpack()[0])
    d = property(lambda self: self._unpack()[1])
    e = property(lambda self: self._unpack()[2])
    tags = property(lambda self: self._unpack()[3] if self.packed is not None
                    else self.tags_dev.cpu().numpy().astype(np.int8))
    perm = property(lambda self: self._unpack()[4] if self.packed is not None
                    else self.perm_dev.cpu().numpy().astype(np.int64))

    def solve(self, B):
        """Solve M X = B (vector or multi-column), factor.py:52-66."""
        device_in = isinstance(B, DeviceArray) or _is_tensor(B)
        one_d = len(B.shape) == 1
        rows = B.shape[0]
        cols = 1 if one_d else (B.shape[1] if len(B.shape) > 1 else 1)
        if rows != self.n:
            raise ValueError(f"rhs has {rows} rows, factor has {self.n}")
        if self.packed is None:
            raise SolverStateError("factor values were released (reduce_domains keep='solution')")
        if self.n == 0 or cols == 0:
            out = np.zeros((self.n, cols), dtype=np.complex128)
            return out[:, 0] if one_d else out
        t = require_cuda()
        Z = to_device(B).reshape(self.n, cols).clone()
        work = empty((self.n, cols))
        if self.n > _lib.PANEL_BK_MIN:
            d_tasks = t.empty(64 * 2 * ((self.n + 63) // 64), dtype=t.uint8, device="cuda")
            _lib.call("d3m_ldlt_solve_blocked_batched", 1, self.n, _P(self.packed), 0, _P(self.perm_dev), 0,
                      _P(self.tags_dev), 0, _P(Z), 0, cols, cols, _P(work), _P(d_tasks), stream_ptr())
        else:
            _lib.call("d3m_ldlt_solve_batched", 1, self.n, _P(self.packed), 0, _P(self.perm_dev), 0,
                      _P(self.tags_dev), 0, _P(Z), 0, cols, cols, _P(work), stream_ptr())
        if one_d:
            Z = Z.reshape(self.n)
        if device_in:
            return DeviceArray(Z)
        del t
        return Z.cpu().numpy()

    def dense_d(self) -> np.ndarray:
        """Block diagonal D as a dense matrix (factor.py:68-80)."""
        _, d, e, tags, _ = self._unpack()
        D = np.diag(d).astype(np.complex128)
        two = np.flatnonzero(tags == 2)
        D[two + 1, two] = e[two]
        D[two, two + 1] = e[two]
        return D


def _is_tensor(x) -> bool:
    return type(x).__module__.startswith("torch")


def dense_ldlt_bk(M, pivot_tol: float = DEFAULT_PIVOT_TOL, margins: bool = False) -> DenseFactor:
    """Bunch-Kaufman LDL^T of a complex symmetric matrix on the GPU.

    factor.py:83-116: rejects non-square input (ValueError), checks symmetry
    to 1e-12 max|M| (ValueError "not symmetric"), raises SingularBlockError
    when neither a 1x1 nor a 2x2 pivot clears pivot_tol * max|M|.  The pivot
    sequence and the factor values are bit-identical to the reference.
    """
    shape = tuple(M.shape) if (isinstance(M, DeviceArray) or _is_tensor(M)) else np.shape(M)
    if len(shape) != 2 or shape[0] != shape[1]:
        raise ValueError("matrix must be square")
    n = int(shape[0])
    t = require_cuda()
    W = to_device(M).clone() if n else t.zeros((0, 0), dtype=t.complex128, device="cuda")
    return _factor_batch(W.reshape(1, n, n), pivot_tol, labels=None, margins=margins)[0]


def _factor_batch(W, pivot_tol, labels, check_sym=True, scratch=None, margins=False):
    """Factor a (batch, n, n) device tensor in place; returns DenseFactors
    or raises for the first failing matrix (``labels`` customises errors)."""
    t = require_cuda()
    batch, n = int(W.shape[0]), int(W.shape[1])
    perm = t.empty((batch, n), dtype=t.int64, device="cuda")
    tags = t.empty((batch, n), dtype=t.int8, device="cuda")
    n2 = t.empty(batch, dtype=t.int32, device="cuda")
    info = t.empty(batch, dtype=t.int32, device="cuda")
    gr = t.empty(batch, dtype=t.float64, device="cuda")
    sc = t.empty(batch, dtype=t.float64, device="cuda")
    asy = t.empty(batch, dtype=t.float64, device="cuda")
    if scratch is None and 64 * n > 200 * 1024:
        scratch = empty((batch, 4 * n))
    mg = t.empty((batch, 2), dtype=t.float64, device="cuda") if margins else None
    _lib.call("d3m_bk_factor_batched", batch, n, _P(W), n * n, max(n, 1), float(pivot_tol), int(check_sym),
              _P(perm), _P(tags), _P(n2), _P(gr), _P(info), _P(sc), _P(asy), _P(scratch), _P(mg), stream_ptr())
    return _collect(W, perm, tags, n2, info, gr, sc, asy, pivot_tol, labels, margin=mg)


def _collect(W, perm, tags, n2, info, gr, sc, asy, pivot_tol, labels, wrap=None, margin=None):
    info_h = info.cpu().numpy()
    sc_h = sc.cpu().numpy()
    bad = np.flatnonzero(info_h != -1)
    if bad.size:
        b = int(bad[0])
        if info_h[b] == -2:
            raise ValueError(f"matrix is not symmetric: max|M - M^T| = {float(asy[b].item()):.3e}")
        msg = _singular_msg(int(info_h[b]), pivot_tol * float(sc_h[b]))
        if wrap is not None:
            raise wrap(b, msg)
        raise SingularBlockError(msg)
    gr_h, n2_h = gr.cpu().numpy(), n2.cpu().numpy()
    facs = [DenseFactor(W[b], perm[b], tags[b], float(gr_h[b]), int(n2_h[b])) for b in range(W.shape[0])]
    if margin is not None:
        for f, mrow in zip(facs, margin.cpu().numpy()):
            f.margin = (float(mrow[0]), float(mrow[1]))
    return facs


# ---------------------------------------------------------------------------
# Block factor
# ---------------------------------------------------------------------------

@dataclass
class FactorStats:
    factor_entries: int = 0
    flops: int = 0
    peak_bytes: int = 0
    growth_factor: float = 1.0
    n_2x2_pivots: int = 0
    # pivot-decision diagnostics (block_ldlt(margins=True); not in the reference)
    decision_margin: float | None = None
    argmax_gap: float | None = None


class _OffDiag(Mapping):
    """Lazy (i, j) -> L_ij mapping over the device panels."""

    def __init__(self, sched, pool):
        self._s = sched
        self._pool = pool
        self._cache = {}

    def __getitem__(self, key):
        if key not in self._s.loc:
            raise KeyError(key)
        if key not in self._cache:
            off, rows, cols = self._s.loc[key]
            self._cache[key] = self._pool[off:off + rows * cols].reshape(rows, cols).cpu().numpy()
        return self._cache[key]

    def device(self, key):
        off, rows, cols = self._s.loc[key]
        return self._pool[off:off + rows * cols].reshape(rows, cols)

    def __iter__(self):
        return iter(self._s.offdiag_keys)

    def __len__(self):
        return len(self._s.offdiag_keys)


class BlockFactor:
    """Output of :func:`block_ldlt` (factor.py:128-136): per-supernode dense
    factors in elimination order, the off-diagonal factor blocks of the
    pattern (lazy host views of the device panels) and statistics."""

    def __init__(self, plan, diag, offdiag, stats, sched=None, pool=None, perm=None, tags=None):
        self.plan = plan
        self.diag = diag
        self.offdiag = offdiag
        self.stats = stats
        self._sched = sched
        self._pool = pool
        self._perm = perm
        self._tags = tags


class _Schedule:
    """Device layout + trailing-update task table of one elimination plan."""

    def __init__(self, plan: EliminationPlan):
        t = require_cuda()
        nb = plan.nblocks
        sizes = np.asarray(plan.sizes_perm, dtype=np.int64)
        self.nb = nb
        self.sizes = sizes
        self.row_off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        pattern = [np.asarray(p, dtype=np.int64) for p in plan.pattern]
        self.pattern = pattern
        self.pat_ptr = np.concatenate([[0], np.cumsum([p.size for p in pattern])]).astype(np.int64)
        self.pat_idx = np.concatenate(pattern).astype(np.int64) if nb and self.pat_ptr[-1] else np.zeros(0, np.int64)
        self.panel_rows = np.array([int(sizes[p].sum()) for p in pattern], dtype=np.int64)
        self.diag_off = np.zeros(nb, dtype=np.int64)
        self.panel_off = np.zeros(nb, dtype=np.int64)
        off = 0
        self.loc = {}               # (i, j) -> (elem offset, rows, cols)
        self.rowpos = {}            # (i, j) -> row offset of block i in panel j
        for j in range(nb):
            nj = int(sizes[j])
            self.diag_off[j] = off
            off += nj * nj
            self.panel_off[j] = off
            r = 0
            for i in pattern[j]:
                i = int(i)
                self.rowpos[(i, j)] = r
                self.loc[(i, j)] = (int(self.panel_off[j]) + r * nj, int(sizes[i]), nj)
                r += int(sizes[i])
            off += int(self.panel_rows[j]) * nj
        self.pool_elems = off
        self.offdiag_keys = sorted(self.loc, key=lambda ij: (ij[1], ij[0]))
        self.piv_elems = int(self.row_off[-1])
        # trailing-update GEMM tasks, "next" (targets in column j+1) first
        # (native planner, csrc/d3m_plan.cpp d3m_plan_gemm_tasks)
        bm = _lib.GEMM_BM
        try:
            tasks, ptr, nxt, tiles_n, tiles_r, self.flops_update = planner.gemm_tasks(
                sizes, pattern, self.diag_off, self.panel_off)
        except ValueError as err:
            raise FactorConsistencyError(str(err)) from None
        self.tasks = tasks
        # panel TRSM as one GEMM per column: X = panel * Binv_j^T
        self.binv_off = np.concatenate([[0], np.cumsum(sizes * sizes)]).astype(np.int64)
        tt = np.zeros(nb, dtype=_lib.GEMM_TASK)
        tt["a_off"] = self.panel_off
        tt["b_off"] = self.binv_off[:nb]
        tt["m"] = self.panel_rows
        tt["n"] = tt["k"] = tt["lda"] = tt["ldb"] = tt["ldc"] = sizes
        # X = (K_panel P^T) L^-T for supernodes <= 512 (d3m_capi.cu kTrsmTriMax): gathered A
        # columns (perm at the column's pivot offset), triangular K range per output tile
        tri = sizes <= _lib.TRSM_TRI_MAX
        tt["flags"] = _lib.GEMM_STORE | np.where(tri, _lib.GEMM_TRIGATHER, 0)
        tt["pad"] = np.where(tri, self.row_off[:nb], 0)
        tt["tiles_n"] = (sizes + bm - 1) // bm
        self.tiles_trsm = (((self.panel_rows + bm - 1) // bm) * ((sizes + bm - 1) // bm)).astype(np.int64)
        self.d_trsm_tasks = upload_bytes(tt)
        self.d_diag_off = upload_i64(self.diag_off if nb else np.zeros(1, np.int64))
        self.d_sizes = upload_i64(sizes if nb else np.zeros(1, np.int64))
        self.part_rows = int(max([len(p) * int(sizes[j]) for j, p in enumerate(pattern)] + [1]))
        self.task_ptr = ptr
        self.task_next = nxt
        self.tiles_next = tiles_n
        self.tiles_rest = tiles_r
        self.d_tasks = upload_bytes(tasks) if len(tasks) else t.zeros(64, dtype=t.uint8, device="cuda")
        # X panels of the columns in flight: a ring of 4 slots (d3m_capi.cu kXSlots)
        self.xbuf_elems = 4 * max(1, int((self.panel_rows * sizes).max()) if nb else 1)
        self.etree_sched = planner.etree_schedule(plan.etree_parent, pattern)
        self.stage_lock = threading.Lock()     # the host-staged upload's pinned ring (one upload at a time)
        # block_solve backward gather: global plan-order rows of every panel
        gidx, gptr = [], [0]
        for j in range(nb):
            for i in pattern[j]:
                gidx.append(np.arange(self.row_off[i], self.row_off[i + 1], dtype=np.int64))
            gptr.append(gptr[-1] + int(self.panel_rows[j]))
        self.gptr = np.asarray(gptr, dtype=np.int64)
        self.d_gidx = upload_i64(np.concatenate(gidx) if gidx else np.zeros(1, np.int64))
        self.flops_trsm = int(sum(4 * int(self.panel_rows[j]) * int(sizes[j]) ** 2 for j in range(nb)))
        self.flops_bk = int(sum(4 * int(s) ** 3 // 3 for s in sizes))     # complex LDL^T: 4n^3/3
        self.stats_cache = {}


_SCHED_CACHE: "OrderedDict[tuple, _Schedule]" = OrderedDict()
_SCHED_LOCK = threading.Lock()
_SCHED_KEEP = 2


def _schedule(plan: EliminationPlan) -> _Schedule:
    """The device layout / task tables of a plan, cached by plan STRUCTURE
    (supernode sizes and block pattern), so a new plan object of the same
    structure (a new solve_d3m run) reuses them; the last _SCHED_KEEP
    structures are kept."""
    sched = getattr(plan, "_d3m_schedule", None)
    key = (tuple(int(s) for s in plan.sizes_perm), tuple(tuple(int(i) for i in p) for p in plan.pattern))
    if sched is not None and sched[0] == key:
        return sched[1]
    with _SCHED_LOCK:
        hit = _SCHED_CACHE.get(key)
        if hit is None:
            hit = _Schedule(plan)
            _SCHED_CACHE[key] = hit
            while len(_SCHED_CACHE) > _SCHED_KEEP:
                _SCHED_CACHE.popitem(last=False)
        else:
            _SCHED_CACHE.move_to_end(key)
    try:
        plan._d3m_schedule = (key, hit)
    except AttributeError:
        pass
    return hit


def _reference_stats(K_keys, sizes_orig, plan: EliminationPlan, inv) -> tuple[int, int, int]:
    """factor_entries, flops and peak_bytes with the reference's bookkeeping
    (factor.py:174-239), evaluated symbolically on the host."""
    sizes = plan.sizes_perm
    live_keys = {}
    for (i, j) in K_keys:
        a, b = int(inv[i]), int(inv[j])
        key = (a, b) if a >= b else (b, a)
        live_keys[key] = int(sizes[key[0]]) * int(sizes[key[1]])
    live = sum(live_keys.values())
    stored = flops = 0
    peak = live
    for j in range(plan.nblocks):
        nj = int(sizes[j])
        if (j, j) in live_keys:
            live -= live_keys.pop((j, j))
        stored += nj * (nj + 1) // 2
        flops += nj ** 3 // 3 + nj ** 2
        rows = [int(r) for r in plan.pattern[j]]
        transient = 0
        for i in rows:
            ni = int(sizes[i])
            if (i, j) in live_keys:
                live -= live_keys.pop((i, j))
            stored += ni * nj
            flops += ni * nj * nj + ni * nj
            transient += ni * nj
        peak = max(peak, live + stored + transient)
        for a, i in enumerate(rows):
            for kk in rows[:a + 1]:
                flops += int(sizes[i]) * nj * int(sizes[kk])
                if (i, kk) not in live_keys:
                    live_keys[(i, kk)] = int(sizes[i]) * int(sizes[kk])
                    live += live_keys[(i, kk)]
        peak = max(peak, live + stored + transient)
    return stored, flops, 16 * peak


def _upload_K(K: BlockSparseSym, sched: _Schedule, plan: EliminationPlan, pool):
    """Copy (and relabel/transpose) the stored blocks of K into the zeroed
    factor pool: factor._permute_blocks (factor.py:139-151) on the device."""
    t = require_cuda()
    inv = plan.order.inverse()
    sizes = K.sizes
    items = []
    for k, b in K.blocks.items():
        # device blocks must be complex128 (the copy kernel reads raw memory):
        # CUDA tensors and DeviceArrays of another dtype are converted first
        if _is_tensor(b) and b.is_cuda:
            b = DeviceArray(to_device(b))
        elif isinstance(b, DeviceArray) and b.tensor.dtype != t.complex128:
            b = DeviceArray(to_device(b))
        items.append((k, b))

    def cpu_view(b):
        return _is_tensor(b) and not b.is_cuda and b.is_contiguous() and b.dtype == t.complex128

    host = [(k, b) for k, b in items if not isinstance(b, DeviceArray) and not cpu_view(b)]
    dev = [(k, b) for k, b in items if isinstance(b, DeviceArray)]
    groups = []          # (src tensor, [(src_off, key, block-shape)])
    # host tensors that are views of one (pinned) allocation: one asynchronous
    # copy of the whole allocation instead of one pageable copy per block
    views: dict[int, tuple] = {}
    for k, b in items:
        if not isinstance(b, DeviceArray) and cpu_view(b):
            base = b.untyped_storage().data_ptr()
            views.setdefault(base, (b, []))[1].append(((b.data_ptr() - base) // 16, k))
    for base, (st, entries) in views.items():
        whole = t.empty(0, dtype=t.complex128).set_(st.untyped_storage(), 0, (st.untyped_storage().nbytes() // 16,))
        dst = empty(int(whole.numel()))
        dst.copy_(whole, non_blocking=bool(whole.is_pinned()))
        groups.append((dst, entries))
    if host:
        tot = sum(int(sizes[i]) * int(sizes[j]) for (i, j), _ in host)
        stage = empty(tot)
        entries, o = [], 0
        for (i, j), b in host:
            nbytes = int(sizes[i]) * int(sizes[j])
            arr = np.ascontiguousarray(np.asarray(b, dtype=np.complex128)).reshape(-1)
            stage[o:o + nbytes].copy_(t.from_numpy(arr))
            entries.append((o, (i, j)))
            o += nbytes
        groups.append((stage, entries))
    if dev:
        bases = {}
        for (i, j), b in dev:
            st = b.tensor
            base = st.untyped_storage().data_ptr()
            bases.setdefault(base, (st, []))[1].append(((st.data_ptr() - base) // 16, (i, j)))
        for base, (st, entries) in bases.items():
            whole = t.empty(0, dtype=t.complex128, device="cuda").set_(st.untyped_storage(), 0,
                                                                        (st.untyped_storage().nbytes() // 16,))
            groups.append((whole, entries))
    for src, entries in groups:
        recs = np.zeros(len(entries), dtype=_lib.COPY_TASK)
        maxe = 1
        for r, (src_off, (i, j)) in enumerate(entries):
            a, b = int(inv[i]), int(inv[j])
            ni, nj = int(sizes[i]), int(sizes[j])
            if a >= b:
                key, transpose = (a, b), 0
            else:
                key, transpose = (b, a), 1
            if key[0] == key[1]:
                dst, ld = int(sched.diag_off[key[0]]), int(plan.sizes_perm[key[0]])
            else:
                if key not in sched.loc:
                    raise FactorConsistencyError(f"block {key} outside the symbolic pattern")
                dst, _, ld = sched.loc[key]
            rows, cols = (ni, nj) if not transpose else (nj, ni)
            recs[r] = (src_off, dst, rows, cols, nj, ld, transpose, _lib.COPY_STORE)
            maxe = max(maxe, rows * cols)
        d_rec = upload_bytes(recs)
        _lib.call("d3m_block_copy", _P(src), _P(pool), _P(d_rec), len(recs), maxe, stream_ptr())
    return groups


_CHUNK_COLS = (2, 4, 8, 16, 24, 32, 48, 64, 96)     # upload chunk boundaries (block columns)


def _first_touch(sched: _Schedule) -> dict:
    """Plan-order block (a, b), a >= b -> the first block column whose BK,
    panel TRSM or trailing update reads or writes it (cached per plan)."""
    ft = getattr(sched, "first_touch", None)
    if ft is None:
        ft = {}
        for j in range(sched.nb):
            pat = [int(i) for i in sched.pattern[j]]
            for key in [(j, j)] + [(i, j) for i in pat] + [(i, k) for a, i in enumerate(pat) for k in pat[:a + 1]]:
                if key not in ft:
                    ft[key] = j
        sched.first_touch = ft
    return ft


def _upload_K_streamed(K: BlockSparseSym, sched: _Schedule, plan: EliminationPlan, pool, flag):
    """Chunked asynchronous upload of K when every block is a view of one
    pinned host allocation: every block (diagonal ones included) goes in the
    chunk of the first block column that touches it (_CHUNK_COLS) on a copy
    stream, each chunk with an event the executor waits on before that column
    (ABI v6), and each chunk flags the exact symmetry of its diagonal blocks
    (ABI v8).  Returns (wait columns, events, keep-alive)
    or None when the inputs do not qualify."""
    t = require_cuda()
    items = list(K.blocks.items())
    # the chunk plan depends only on the block layout: cached per schedule,
    # keyed by every block's key and host address (repeated factorisations of
    # one pinned K skip the validation and the record building, ~4 ms)
    try:
        sig = tuple((k, b.data_ptr()) for k, b in items)
    except AttributeError:
        return None
    cache = getattr(sched, "upload_cache", None)
    if cache is None:
        cache = sched.upload_cache = {}
    hit = cache.get(sig)
    if hit is not None:
        base, recs, d_rec, plan_chunks, o, kentries = hit
        return _stream_chunks(sched, pool, flag, base, recs, d_rec, plan_chunks, o, kentries)
    base = None
    for _, b in items:
        if not (_is_tensor(b) and not b.is_cuda and b.is_contiguous() and b.dtype == t.complex128 and b.is_pinned()):
            return None
        bb = b.untyped_storage().data_ptr()
        if base is None:
            base = bb
        elif bb != base:
            return None
    if base is None:
        return None
    nb = plan.nblocks
    inv = plan.order.inverse()
    sizes = K.sizes
    ft = _first_touch(sched)
    bounds = [0] + [c for c in _CHUNK_COLS if c < nb] + [nb]
    chunks = [[] for _ in range(len(bounds) - 1)]
    for (i, j), b in items:
        a, c = int(inv[i]), int(inv[j])
        key = (a, c) if a >= c else (c, a)
        if key not in ft:
            raise FactorConsistencyError(f"block {key} outside the symbolic pattern")
        ch = int(np.searchsorted(bounds, ft[key], side="right")) - 1
        chunks[ch].append(((i, j), b))
    recs = np.zeros(len(items), dtype=_lib.COPY_TASK)
    plan_chunks, r, o = [], 0, 0
    kentries = []                          # (offset in stage, original key): K stays in stage
    for ch, entries in enumerate(chunks):
        if not entries:
            continue
        r0, maxe = r, 1
        doff, soff, nby, diag = [], [], [], []
        for (i, j), b in entries:
            a, c = int(inv[i]), int(inv[j])
            ni, nj = int(sizes[i]), int(sizes[j])
            key, transpose = ((a, c), 0) if a >= c else ((c, a), 1)
            if key[0] == key[1]:
                dst, ld = int(sched.diag_off[key[0]]), int(plan.sizes_perm[key[0]])
                diag.append(key[0])
            else:
                dst, _, ld = sched.loc[key]
            rows, cols = (ni, nj) if not transpose else (nj, ni)
            recs[r] = (o, dst, rows, cols, nj, ld, transpose, _lib.COPY_STORE)
            kentries.append((o, (i, j)))
            maxe = max(maxe, rows * cols)
            doff.append(16 * o)
            soff.append(b.data_ptr() - base)
            nby.append(16 * ni * nj)
            o += ni * nj
            r += 1
        plan_chunks.append((bounds[ch], r0, r - r0, maxe, np.asarray(doff, np.int64), np.asarray(soff, np.int64),
                            np.asarray(nby, np.int64), upload_i64(np.asarray(diag, np.int64)) if diag else None,
                            len(diag)))
    d_rec = upload_bytes(recs)
    if len(cache) >= 4:
        cache.clear()
    cache[sig] = (base, recs, d_rec, plan_chunks, o, kentries)
    return _stream_chunks(sched, pool, flag, base, recs, d_rec, plan_chunks, o, kentries)


def _stream_chunks(sched, pool, flag, base, recs, d_rec, plan_chunks, o, kentries):
    """Issue the chunked upload planned by _upload_K_streamed on the copy stream."""
    t = require_cuda()
    nb = sched.nb
    stage = empty(max(o, 1))
    cur = t.cuda.current_stream()
    cs = getattr(sched, "copy_stream", None)
    if cs is None:
        cs = sched.copy_stream = t.cuda.Stream()
    ready = t.cuda.Event()
    ready.record(cur)                      # pool zeroed, flag / staging allocated
    cs.wait_event(ready)
    csp = _lib.ctypes.c_void_p(cs.cuda_stream)
    H = _lib.hptr
    waits, events = [], []
    for n, (col, r0, cnt, maxe, doff, soff, nby, d_diag, ndiag) in enumerate(plan_chunks):
        _lib.call("d3m_memcpy_batch", _P(stage), _lib.ctypes.c_void_p(base), H(doff), H(soff), H(nby), cnt, 1, csp)
        _lib.call("d3m_block_copy", _P(stage), _P(pool), _lib.ctypes.c_void_p(d_rec.data_ptr() + r0 * recs.itemsize),
                  cnt, maxe, csp)
        if ndiag:                          # exact-symmetry flags of the chunk's diagonal blocks (as uploaded)
            _lib.call("d3m_diag_sym_flags", _P(pool), _P(sched.d_diag_off), _P(sched.d_sizes), _P(d_diag), ndiag,
                      _P(flag), csp)
        ev = t.cuda.Event()
        ev.record(cs)
        if n == 0:
            cur.wait_event(ev)             # the first columns' blocks and flags
        else:
            waits.append(col)
            events.append(ev)
    stage.record_stream(cs)
    d_rec.record_stream(cs)
    return np.asarray(waits, dtype=np.int64), events, (stage, d_rec), [(stage, kentries)]


def _host_layout(K: BlockSparseSym, sched: _Schedule, plan: EliminationPlan):
    """Chunk layout of a host-staged upload (_upload_K_hoststaged): cached per
    schedule and block-key set.  Blocks go in the chunk of the first block
    column that touches them (_CHUNK_COLS), in staging order; returns
    (keys, copy records, device records, chunks, staged elements, kentries)
    with chunks = [(first column, record start, count, max entries,
    item indices, staging offsets, diag device array, diag count)]."""
    keys = tuple(K.blocks)
    cache = getattr(sched, "host_layout", None)
    if cache is None:
        cache = sched.host_layout = {}
    hit = cache.get(keys)
    if hit is not None:
        return hit
    nb = plan.nblocks
    inv = plan.order.inverse()
    sizes = K.sizes
    ft = _first_touch(sched)
    bounds = [0] + [c for c in _CHUNK_COLS if c < nb] + [nb]
    chunks = [[] for _ in range(len(bounds) - 1)]
    for idx, (i, j) in enumerate(keys):
        a, c = int(inv[i]), int(inv[j])
        key = (a, c) if a >= c else (c, a)
        if key not in ft:
            raise FactorConsistencyError(f"block {key} outside the symbolic pattern")
        chunks[int(np.searchsorted(bounds, ft[key], side="right")) - 1].append(idx)
    recs = np.zeros(len(keys), dtype=_lib.COPY_TASK)
    out_chunks, r, o, kentries = [], 0, 0, []
    for ch, members in enumerate(chunks):
        if not members:
            continue
        r0, maxe, offs, diag = r, 1, [], []
        for idx in members:
            i, j = keys[idx]
            a, c = int(inv[i]), int(inv[j])
            ni, nj = int(sizes[i]), int(sizes[j])
            key, transpose = ((a, c), 0) if a >= c else ((c, a), 1)
            if key[0] == key[1]:
                dst, ld = int(sched.diag_off[key[0]]), int(plan.sizes_perm[key[0]])
                diag.append(key[0])
            else:
                dst, _, ld = sched.loc[key]
            rows, cols = (ni, nj) if not transpose else (nj, ni)
            recs[r] = (o, dst, rows, cols, nj, ld, transpose, _lib.COPY_STORE)
            kentries.append((o, (i, j)))
            maxe = max(maxe, rows * cols)
            offs.append(o)
            o += ni * nj
            r += 1
        out_chunks.append((bounds[ch], r0, r - r0, maxe, members, offs,
                           upload_i64(np.asarray(diag, np.int64)) if diag else None, len(diag)))
    hit = (keys, recs, upload_bytes(recs), out_chunks, o, kentries)
    if len(cache) >= 4:
        cache.clear()
    cache[keys] = hit
    return hit


def _host_stageable(K: BlockSparseSym) -> bool:
    """All blocks on the host (numpy arrays or CPU tensors): the host-staged upload applies."""
    items = list(K.blocks.values())
    return bool(items) and not any(isinstance(b, DeviceArray) or (_is_tensor(b) and b.is_cuda) for b in items)


def _upload_K_hoststaged(K: BlockSparseSym, sched: _Schedule, plan: EliminationPlan, pool, flag):
    """Chunked upload of K from pageable host arrays (numpy blocks, as the
    reference API takes them).  A native host thread (d3m_host_stage_start)
    copies chunk after chunk into a pinned staging buffer, cached on the
    schedule, and publishes each chunk through a pinned flag; the copy stream
    holds each chunk's H2D copy until its flag (d3m_stream_wait_flag), so the
    first columns' factorisation starts while the host is still staging the
    later blocks.  The host thread starts before the waits are enqueued, so
    blocking launches (CUDA_LAUNCH_BLOCKING=1, profilers) cannot deadlock.
    Returns (wait columns, events, keep-alive, kgroups, handle); the caller
    holds sched.stage_lock until the join."""
    t = require_cuda()
    items = list(K.blocks.items())
    keys, recs, d_rec, chunks, o, kentries = _host_layout(K, sched, plan)
    # sources: C-contiguous complex128 host arrays, alive until the join
    src = []
    for _, b in items:
        a = b.numpy() if _is_tensor(b) else b
        src.append(np.ascontiguousarray(np.asarray(a, dtype=np.complex128)))
    for (i, j), a in zip(keys, src):
        if a.size != int(K.sizes[i]) * int(K.sizes[j]):
            raise ValueError(f"block {(i, j)} has shape {a.shape}, expected {(int(K.sizes[i]), int(K.sizes[j]))}")
    prev = getattr(sched, "pin_busy", None)
    if prev is not None:
        prev.synchronize()                 # the last upload's copies out of the staging buffer are done
    pin = getattr(sched, "pin_stage", None)
    if pin is None or pin.numel() < o:
        pin = sched.pin_stage = t.empty(max(o, 1), dtype=t.complex128, pin_memory=True)
        sched.pin_flag = t.zeros(1, dtype=t.int32, pin_memory=True)
    pflag = sched.pin_flag
    pflag.numpy()[0] = 0
    H = _lib.hptr
    fptr = _lib.ctypes.c_void_p(pflag.data_ptr())
    chunk_ptr, order, dst_off, nbytes = [0], [], [], []
    for (col, r0, cnt, maxe, members, offs, d_diag, ndiag) in chunks:
        for m, off in zip(members, offs):
            order.append(m)
            dst_off.append(16 * off)
            nbytes.append(16 * src[m].size)
        chunk_ptr.append(len(order))
    srcp = (_lib.ctypes.c_void_p * max(len(order), 1))(*[src[m].ctypes.data for m in order])
    handle = _lib.load().d3m_host_stage_start(len(chunks), H(np.asarray(chunk_ptr, np.int64)), len(order), srcp,
                                              H(np.asarray(dst_off, np.int64)), H(np.asarray(nbytes, np.int64)),
                                              _lib.ctypes.c_void_p(pin.data_ptr()), fptr,
                                              min(8, _os.cpu_count() or 1))
    if not handle:
        raise _lib.D3MError("d3m_host_stage_start failed")
    handle = _lib.ctypes.c_void_p(handle)
    try:
        stage = empty(max(o, 1))
        cur = t.cuda.current_stream()
        cs = getattr(sched, "copy_stream", None)
        if cs is None:
            cs = sched.copy_stream = t.cuda.Stream()
        ready = t.cuda.Event()
        ready.record(cur)                  # pool zeroed, flag / staging allocated
        cs.wait_event(ready)
        csp = _lib.ctypes.c_void_p(cs.cuda_stream)
        waits, events = [], []
        for n, (col, r0, cnt, maxe, members, offs, d_diag, ndiag) in enumerate(chunks):
            lo, hi = offs[0], offs[-1] + src[members[-1]].size
            _lib.call("d3m_stream_wait_flag", fptr, n + 1, csp)
            _lib.call("d3m_memcpy_batch", _P(stage), _lib.ctypes.c_void_p(pin.data_ptr()),
                      H(np.array([16 * lo], np.int64)), H(np.array([16 * lo], np.int64)),
                      H(np.array([16 * (hi - lo)], np.int64)), 1, 1, csp)
            _lib.call("d3m_block_copy", _P(stage), _P(pool),
                      _lib.ctypes.c_void_p(d_rec.data_ptr() + r0 * recs.itemsize), cnt, maxe, csp)
            if ndiag:                      # exact-symmetry flags of the chunk's diagonal blocks (as uploaded)
                _lib.call("d3m_diag_sym_flags", _P(pool), _P(sched.d_diag_off), _P(sched.d_sizes), _P(d_diag), ndiag,
                          _P(flag), csp)
            ev = t.cuda.Event()
            ev.record(cs)
            if n == 0:
                cur.wait_event(ev)         # the first columns' blocks and flags
            else:
                waits.append(col)
                events.append(ev)
        sched.pin_busy = events[-1] if events else ev
        stage.record_stream(cs)
        d_rec.record_stream(cs)
    except BaseException:
        _lib.load().d3m_host_stage_join(handle)
        raise
    return (np.asarray(waits, dtype=np.int64), events, (stage, d_rec, src, pin), [(stage, kentries)], handle)


def block_ldlt(K: BlockSparseSym, plan: EliminationPlan, pivot_tol: float = DEFAULT_PIVOT_TOL,
               lookahead: bool = True, margins: bool = False) -> BlockFactor:
    """Right-looking block LDL^T of ``K`` following ``plan`` on one GPU.

    factor.py:154-240: per block column j, Bunch-Kaufman of the diagonal
    block (bit-exact kernel), X_ij = L_ij D_jj by a triangular solve against
    every pattern row, L_ij = X_ij D_jj^-1, then K_ik -= X_ij L_kj^T for
    pattern pairs i >= k on the DMMA tensor pipe (diagonal targets
    symmetrised from the lower half).  The next column's factorisation
    overlaps the current column's trailing update (lookahead).

    ``margins`` (an extension; the reference has no such output) tracks the
    pivot-decision margins of every diagonal block: each DenseFactor gets
    ``margin`` = (decision margin, argmax gap) and ``stats`` the minima over
    the blocks (FactorStats.decision_margin / argmax_gap).
    """
    nb = K.nblocks
    if plan.nblocks != nb:
        raise ValueError("plan and matrix disagree on block count")
    t = require_cuda()
    inv = plan.order.inverse()
    if nb == 0:
        return BlockFactor(plan, [], {}, FactorStats(0, 0, 0, 1.0, 0))
    sched = _schedule(plan)
    keyset = frozenset(K.blocks)
    if keyset not in sched.stats_cache:
        sched.stats_cache[keyset] = _reference_stats(list(K.blocks), K.sizes, plan, inv)
    stored, flops, peak = sched.stats_cache[keyset]
    pool = empty(max(sched.pool_elems, 1))
    _lib.call("d3m_zero", _P(pool), sched.pool_elems, stream_ptr())
    # exactly symmetric diagonal blocks stay exactly symmetric (mirrored SYM
    # updates): the diagonal BK then needs only the lower triangle
    # per-block exact-symmetry flags (2: bitwise symmetric, the BK reads the
    # lower triangle only; 1: full check), read by each column's BK on the
    # device (ABI v8): no host sync on the upload of K's diagonal
    flag = t.ones(max(nb, 1), dtype=t.int32, device="cuda")
    streamed = _upload_K_streamed(K, sched, plan, pool, flag)
    stage_handle = None
    staged = False
    if streamed is None and _host_stageable(K):
        # the plan's pinned staging ring and flag serve one upload at a time
        # (another thread factoring with the same plan waits here)
        sched.stage_lock.acquire()
        staged = True
        try:
            *streamed, stage_handle = _upload_K_hoststaged(K, sched, plan, pool, flag)
        except BaseException:
            sched.stage_lock.release()
            raise
    try:
        return _block_ldlt_run(K, plan, pivot_tol, lookahead, margins, sched, pool, flag, streamed, stored, flops,
                               peak, inv)
    finally:
        try:
            if stage_handle is not None:   # the host thread reads the caller's arrays until here
                _lib.call("d3m_host_stage_join", stage_handle)
        finally:
            if staged:
                sched.stage_lock.release()


def _block_ldlt_run(K, plan, pivot_tol, lookahead, margins, sched, pool, flag, streamed, stored, flops, peak, inv):
    t = require_cuda()
    nb = K.nblocks
    if streamed is None:
        kgroups = _upload_K(K, sched, plan, pool)
        if getattr(sched, "d_all_blocks", None) is None:
            sched.d_all_blocks = upload_i64(np.arange(nb, dtype=np.int64))
        _lib.call("d3m_diag_sym_flags", _P(pool), _P(sched.d_diag_off), _P(sched.d_sizes), _P(sched.d_all_blocks), nb,
                  _P(flag), stream_ptr())
        wait_cols, wait_ev = np.zeros(1, np.int64), np.zeros(1, np.uint64)
        nwait = 0
    else:
        wait_cols, events, _keep, kgroups = streamed
        nwait = len(events)
        wait_ev = np.asarray([e.cuda_event for e in events] or [0], dtype=np.uint64)
        if nwait == 0:
            wait_cols = np.zeros(1, np.int64)
    check_sym = 1                          # superseded per block by the device flags
    perm = t.empty(max(sched.piv_elems, 1), dtype=t.int64, device="cuda")
    tags = t.empty(max(sched.piv_elems, 1), dtype=t.int8, device="cuda")
    info = t.empty(nb, dtype=t.int32, device="cuda")
    n2 = t.empty(nb, dtype=t.int32, device="cuda")
    gr = t.empty(nb, dtype=t.float64, device="cuda")
    sc = t.empty(nb, dtype=t.float64, device="cuda")
    asy = t.empty(nb, dtype=t.float64, device="cuda")
    xbuf = empty(sched.xbuf_elems)
    binv = empty(max(int(sched.binv_off[-1]), 1))
    nmax = int(sched.sizes.max())
    scratch = empty(4 * 4 * nmax) if 64 * nmax > 200 * 1024 else None      # one per critical stream
    mg = t.empty((nb, 2), dtype=t.float64, device="cuda") if margins else None
    H = _lib.hptr
    _lib.call("d3m_block_ldlt_exec", nb, H(sched.sizes), H(sched.diag_off), H(sched.panel_off),
              H(sched.panel_rows), H(sched.row_off), H(sched.binv_off), H(sched.task_ptr), H(sched.task_next),
              H(sched.tiles_next), H(sched.tiles_rest), H(sched.tiles_trsm), _P(sched.d_tasks),
              _P(sched.d_trsm_tasks), _P(pool), _P(binv), _P(xbuf), sched.xbuf_elems, _P(perm), _P(tags),
              _P(info), _P(n2), _P(gr), _P(sc), _P(asy), _P(scratch), float(pivot_tol), check_sym,
              int(bool(lookahead)), nwait, H(wait_cols), H(wait_ev), _P(flag), _P(mg), H(sched.etree_sched),
              stream_ptr())
    info_h = info.cpu().numpy()
    bad = np.flatnonzero(info_h != -1)
    if bad.size:
        j = int(bad[0])
        if info_h[j] == -2:
            raise ValueError(f"matrix is not symmetric: max|M - M^T| = {float(asy[j].item()):.3e}")
        err = SingularBlockError(_singular_msg(int(info_h[j]), pivot_tol * float(sc[j].item())))
        raise SingularBlockError(f"block column {j}: {err}") from err
    gr_h, n2_h = gr.cpu().numpy(), n2.cpu().numpy()
    diag = []
    for j in range(nb):
        nj = int(sched.sizes[j])
        o, r = int(sched.diag_off[j]), int(sched.row_off[j])
        diag.append(DenseFactor(pool[o:o + nj * nj].reshape(nj, nj), perm[r:r + nj], tags[r:r + nj],
                                float(gr_h[j]), int(n2_h[j])))
    stats = FactorStats(stored, flops, peak, float(max(gr_h.max(), 1.0)) if nb else 1.0, int(n2_h.sum()))
    stats.growth_factor = float(max((f.growth for f in diag), default=1.0))
    if mg is not None:
        mh = mg.cpu().numpy()
        for f, mrow in zip(diag, mh):
            f.margin = (float(mrow[0]), float(mrow[1]))
        stats.decision_margin, stats.argmax_gap = float(mh[:, 0].min()), float(mh[:, 1].min())
    F = BlockFactor(plan, diag, _OffDiag(sched, pool), stats, sched, pool, perm, tags)
    F._binv = binv
    # device copy of K's stored blocks (the upload staging buffer or the
    # caller's device blocks), kept for block_solve(refine=...)
    F._kgroups = kgroups
    F._ksizes = np.asarray(K.sizes, dtype=np.int64)
    return F


def _solve_plan(sched: _Schedule):
    """Device copy of the plan arrays for the persistent block solve (ABI v5,
    include/d3m.h d3m_block_solve_exec), built once per plan."""
    if getattr(sched, "d_solve_plan", None) is None:
        nb = sched.nb
        arr = np.concatenate([sched.sizes, sched.row_off[:nb], sched.diag_off, sched.panel_off, sched.panel_rows,
                              sched.row_off[:nb], sched.binv_off[:nb], sched.gptr]).astype(np.int64)
        sched.d_solve_plan = upload_i64(arr)
    return sched.d_solve_plan


_FA, _FD, _FB, _BC, _BR, _BE = 0, 1, 2, 3, 4, 5      # skinny_dmma.cu FlowItem types
_KCH = 256                                            # backward split-K chunk (panel rows)
_FD_ROWS, _BR_ROWS = 32, 16                           # rows per D^-1 / reduce work item


def _solve_flow(sched: _Schedule):
    """Work-item list of the dataflow block solve (include/d3m.h
    d3m_block_solve_dataflow), built once per plan.

    The items are the barrier kernel's tiles; their order is a topological
    order that puts each column's critical items first: forward, after
    z_j (FA) come the updates of the parent block (first pattern block) and
    only then the previous column's updates of farther blocks; backward, the
    partials of the chunks holding the parent block come before the reduce
    and the Binv^T tiles, the farther chunks of column j-1 right after.
    Updates of one 16-row tile stay in ascending column order (per-tile
    sequence counters), as in the barrier kernel's phases.

    The list is then split (``chain_split``): the critical chain first (its
    own queue, run by CTAs that own their SM), the rest after, each part in
    this order.  Returns (items, nitems, nchain, deps, part_off, counter
    count incl. the scheduler scratch, partial elements)."""
    fl = getattr(sched, "flow", None)
    if fl is None:
        it, dp, part_off, ncnt, part_elems = flow_items(sched.sizes, sched.pattern, sched.panel_rows)
        it, nchain = chain_split(it, sched.sizes, sched.pattern)
        fl = sched.flow = (upload_bytes(it), len(it), nchain, upload_bytes(dp), upload_i64(part_off),
                           ncnt + _lib.FLOW_EXTRA_COUNTERS, part_elems)
    return fl


def chain_split(items, sizes, pattern):
    """(items reordered: critical chain first, nchain).  Chain items: z_j
    (FA), the reduce and x_j (BR, BE), the updates of the parent block's
    rows (FB with panel row < n_parent; the parent is the first pattern
    block) and the partials of the chunks holding them (BC with 256 chunk <
    n_parent).  D^-1 (FD, needed only by the backward sweep) and the farther
    updates / partials run on the other CTAs.  Stable: each part keeps the
    planner's topological order."""
    items = np.asarray(items)
    nb = len(sizes)
    npar = np.array([int(sizes[int(p[0])]) if len(p) else 0 for p in pattern] + [0], dtype=np.int64)
    typ, j, p0 = items[:, 0], items[:, 1], items[:, 2].astype(np.int64)
    jn = np.where((j >= 0) & (j < nb), j, nb)
    crit = ((typ == _FA) | (typ == _BR) | (typ == _BE) | ((typ == _FB) & (p0 < npar[jn]))
            | ((typ == _BC) & (p0 * _KCH < npar[jn])))
    order = np.concatenate([np.nonzero(crit)[0], np.nonzero(~crit)[0]])
    return np.ascontiguousarray(items[order]), int(crit.sum())


def flow_items(sizes, pattern, panel_rows):
    """Work list of the dataflow block solve, built by the native planner
    (csrc/d3m_plan.cpp d3m_plan_flow_items; tests/test_solve_flow.py checks
    it is a topological order and equals the Python restatement).  Returns
    (items int32 [n, 8], deps int32 [m, 2], part_off int64 [nb], counter
    count, partial elems)."""
    return planner.flow_items(sizes, pattern, panel_rows)


def _residual_launches(F: BlockFactor, cols: int):
    """Grouped-GEMM launches computing r -= K x over K's stored blocks
    (include/d3m.h d3m_block_residual), cached per block layout and RHS count.

    Stored block (i, j) contributes K_ij x_j to row block i and, off the
    diagonal, K_ij^T x_i to row block j (blockmat.py:93-101's symmetric
    scatter).  Contributions to one target are ordered by (source, term) and
    launch round t carries every target's t-th contribution, so no two tasks
    of a launch write the same rows and the sum order is fixed."""
    sched, plan = F._sched, F.plan
    # the task records depend only on the block layout (groups' entries) and
    # the RHS count: cached per schedule; the groups' base pointers are
    # refreshed per factor (a new upload staging buffer each call)
    cache = getattr(sched, "res_cache", None)
    if cache is None:
        cache = sched.res_cache = {}
    key = (cols, tuple(tuple(e) for _, e in F._kgroups))
    hit = cache.get(key)
    if hit is not None:
        nl, ta, nt, tiles, toff, gidx, d_tasks = hit
        base = np.asarray([F._kgroups[g][0].data_ptr() for g in gidx], np.uint64)
        return nl, ta, nt, tiles, toff, base, d_tasks
    inv = plan.order.inverse()
    ks = F._ksizes
    row_off = sched.row_off
    per_target: dict[int, list] = {}
    for gi, (src, entries) in enumerate(F._kgroups):
        for off, (i, j) in entries:
            a, c = int(inv[i]), int(inv[j])
            ni, nj = int(ks[i]), int(ks[j])
            per_target.setdefault(a, []).append((c, 0, gi, int(off), ni, nj, 0, nj))
            if i != j:
                per_target.setdefault(c, []).append((a, 1, gi, int(off), nj, ni, 1, nj))
    rounds: dict[tuple, list] = {}
    for a, lst in per_target.items():
        for t, (c, term, gi, off, m, k, ta, lda) in enumerate(sorted(lst)):
            rounds.setdefault((t, gi, ta), []).append((a, c, off, m, k, lda))
    recs, ta_l, nt_l, tiles_l, off_l, base_l, g_l = [], [], [], [], [], [], []
    for (t, gi, ta) in sorted(rounds):
        lst = rounds[(t, gi, ta)]
        rec = np.zeros(len(lst), dtype=_lib.GEMM_TASK)
        tiles = 0
        for r_, (a, c, off, m, k, lda) in enumerate(lst):
            tn = (cols + _lib.GEMM_BN - 1) // _lib.GEMM_BN
            rec[r_] = (off, int(row_off[c]) * cols, int(row_off[a]) * cols, m, cols, k, lda, cols, cols,
                       _lib.GEMM_SUB, tiles, tn, 0)
            tiles += ((m + _lib.GEMM_BM - 1) // _lib.GEMM_BM) * tn
        off_l.append(sum(len(x) for x in recs))
        recs.append(rec)
        ta_l.append(ta)
        nt_l.append(len(lst))
        tiles_l.append(tiles)
        base_l.append(F._kgroups[gi][0].data_ptr())
        g_l.append(gi)
    d_tasks = upload_bytes(np.concatenate(recs))
    arrs = (len(recs), np.asarray(ta_l, np.int32), np.asarray(nt_l, np.int32), np.asarray(tiles_l, np.int32),
            np.asarray(off_l, np.int64))
    if len(cache) >= 8:
        cache.clear()
    cache[key] = arrs + (g_l, d_tasks)
    return arrs + (np.asarray(base_l, np.uint64), d_tasks)


def block_solve(F: BlockFactor, g: list, refine: int = 0) -> list:
    """Solve K x = g through the block factor (factor.py:271-310).

    ``g`` is a block vector in the original block numbering, each block 1-D
    or a matrix of RHS columns.  All columns go through one device pass, each
    computed independently, so k-RHS results equal k single solves bit for
    bit.  Device-resident inputs give device-resident outputs; host torch
    tensors give host torch tensors (views of one pinned copy), numpy gives
    numpy.

    ``refine`` (not in the reference, default 0 = the reference's algorithm):
    steps of fixed-precision iterative refinement, x += solve(g - K x), with
    K x formed on the tensor pipe from the device copy of K's stored blocks
    that block_ldlt keeps.  One step takes the relative residual of config 4
    from ~4e-10 (the reference's own: ~1e-10) to rounding level.
    """
    nb = F.plan.nblocks
    if len(g) != nb:
        raise ValueError(f"block vector has {len(g)} blocks, expected {nb}")
    if nb == 0:
        return []
    perm = F.plan.order.perm
    sizes = F.plan.sizes_perm
    # host torch tensors (e.g. pinned RHS) take the host path and get host
    # tensors back: one staged H2D copy in, one D2H copy out
    cpu_t = all(_is_tensor(b) and not b.is_cuda for b in g)
    device_in = not cpu_t and all(isinstance(b, DeviceArray) or _is_tensor(b) for b in g)
    shapes = [tuple(b.shape) for b in g]
    one_d = all(len(s) == 1 for s in shapes)
    cols = None
    for s in shapes:
        c = 1 if len(s) == 1 else s[1]
        if cols is None:
            cols = c
        elif c != cols:
            raise ValueError("inconsistent RHS column counts across blocks")
    for j in range(nb):
        if shapes[int(perm[j])][0] != int(sizes[j]):
            raise ValueError(f"block {int(perm[j])} has wrong length")
    sched = F._sched
    t = require_cuda()
    N = int(sched.row_off[-1])
    if cols == 0:
        out = [np.zeros((int(s[0]), 0), dtype=np.complex128) for s in shapes]
        return out
    if device_in:
        parts = [to_device(g[int(perm[j])]).reshape(int(sizes[j]), cols) for j in range(nb)]
        b = t.cat(parts, dim=0).contiguous()
    elif cpu_t:
        hp = t.empty((N, cols), dtype=t.complex128, pin_memory=True)
        host = hp.numpy()
        for j in range(nb):
            host[sched.row_off[j]:sched.row_off[j + 1]] = g[int(perm[j])].numpy().reshape(int(sizes[j]), cols)
        b = hp.to("cuda", non_blocking=True)
    else:
        host = np.empty((N, cols), dtype=np.complex128)
        for j in range(nb):
            blk = np.asarray(g[int(perm[j])], dtype=np.complex128).reshape(int(sizes[j]), cols)
            host[sched.row_off[j]:sched.row_off[j + 1]] = blk
        b = to_device(host)
    u = empty((N, cols))
    x = empty((N, cols))
    H = _lib.hptr
    if _SOLVE_MODE == "flow":
        # dataflow kernel: per-column partial storage, counters
        d_items, nitems, nchain, d_deps, d_poff, ncnt, part_elems = _solve_flow(sched)
        part = empty(part_elems)
        counters = t.empty(ncnt, dtype=t.int32, device="cuda")

        def solve(rhs, out):
            _lib.call("d3m_block_solve_dataflow", nb, _P(_solve_plan(sched)), _P(d_items), nitems, nchain, _P(d_deps),
                      _P(d_poff), _P(counters), ncnt, _P(sched.d_gidx), _P(F._pool), _P(F._binv), _P(F._tags),
                      _P(rhs), _P(u), _P(out), _P(part), int(cols), stream_ptr())
    else:
        tmp = empty((int(sched.sizes.max()), cols))
        # split-K partials of the backward L^T x products: ceil(R_j / 256) chunks x n_j x 16 RHS (one pass)
        part_elems = int(max(((int(r) + 255) // 256) * int(n) for r, n in zip(sched.panel_rows, sched.sizes))) * 16
        part = empty(max(part_elems, 1))

        def solve(rhs, out):
            _lib.call("d3m_block_solve_exec", nb, H(sched.sizes), H(sched.row_off), H(sched.diag_off),
                      H(sched.panel_off), H(sched.panel_rows), H(sched.row_off), H(sched.binv_off), H(sched.gptr),
                      _P(sched.d_gidx), _P(F._pool), _P(F._binv), _P(F._tags), _P(rhs), _P(u), _P(out), _P(tmp),
                      _P(part), part_elems, int(cols), _P(_solve_plan(sched)), stream_ptr())

    if refine:
        if getattr(F, "_kgroups", None) is None:
            raise SolverStateError("block_solve(refine=...) needs the factor's copy of K (block_ldlt output)")
        b0 = empty((N, cols))
        b0.copy_(b)                   # the solve consumes its right-hand side in place
    solve(b, x)
    if refine:
        nl, ta, nt, tiles, toff, base, d_tasks = _residual_launches(F, int(cols))
        r, d = empty((N, cols)), empty((N, cols))
        add = np.zeros(1, dtype=_lib.COPY_TASK)
        add[0] = (0, 0, N, cols, cols, cols, 0, _lib.COPY_ADD)
        d_add = upload_bytes(add)
        for _ in range(int(refine)):
            r.copy_(b0)
            _lib.call("d3m_block_residual", nl, H(ta), H(nt), H(tiles), H(toff), H(base), _P(x), _P(r),
                      _P(d_tasks), stream_ptr())
            solve(r, d)
            _lib.call("d3m_block_copy", _P(d), _P(x), _P(d_add), 1, N * cols, stream_ptr())
    out = [None] * nb
    if device_in:
        for j in range(nb):
            blk = x[sched.row_off[j]:sched.row_off[j + 1]]
            out[int(perm[j])] = DeviceArray(blk[:, 0] if one_d else blk)
        return out
    if cpu_t:
        xo = t.empty((N, cols), dtype=t.complex128, pin_memory=True)
        xo.copy_(x)                                   # one D2H copy (synchronous: the result is ready)
        for j in range(nb):
            blk = xo[int(sched.row_off[j]):int(sched.row_off[j + 1])]
            out[int(perm[j])] = blk[:, 0] if one_d else blk
        return out
    xh = x.cpu().numpy()
    for j in range(nb):
        blk = xh[sched.row_off[j]:sched.row_off[j + 1]]
        out[int(perm[j])] = blk[:, 0].copy() if one_d else blk.copy()
    return out


def to_device_blocks(K: BlockSparseSym) -> BlockSparseSym:
    """Copy of K whose blocks are views into ONE device pool (one H2D copy),
    the layout block_ldlt consumes with a single relabel/copy launch."""
    t = require_cuda()
    keys = list(K.blocks)
    offs, tot = [], 0
    for (i, j) in keys:
        offs.append(tot)
        tot += int(K.sizes[i]) * int(K.sizes[j])
    host = t.empty(max(tot, 1), dtype=t.complex128, pin_memory=True)
    hv = host.numpy()
    for (i, j), o in zip(keys, offs):
        hv[o:o + int(K.sizes[i]) * int(K.sizes[j])] = np.asarray(K.blocks[(i, j)], dtype=np.complex128).reshape(-1)
    pool = host.to("cuda", non_blocking=False)
    out = BlockSparseSym(K.sizes)
    for (i, j), o in zip(keys, offs):
        ni, nj = int(K.sizes[i]), int(K.sizes[j])
        out.blocks[(i, j)] = DeviceArray(pool[o:o + ni * nj].reshape(ni, nj))
    out._d3m_pool = pool
    return out


def scatter_factor(F: BlockFactor) -> tuple[np.ndarray, np.ndarray]:
    """Dense (L, D) of the permuted matrix, for verification (factor.py:313-334)."""
    sizes = F.plan.sizes_perm
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    n = int(off[-1])
    L = np.zeros((n, n), dtype=np.complex128)
    D = np.zeros((n, n), dtype=np.complex128)
    for j in range(F.plan.nblocks):
        fac = F.diag[j]
        lb = np.zeros_like(fac.L)
        lb[fac.perm, :] = fac.L
        L[off[j]:off[j + 1], off[j]:off[j + 1]] = lb
        D[off[j]:off[j + 1], off[j]:off[j + 1]] = fac.dense_d()
        for i in F.plan.pattern[j]:
            i = int(i)
            L[off[i]:off[i + 1], off[j]:off[j + 1]] = F.offdiag[(i, j)]
    return L, D

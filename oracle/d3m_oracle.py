"""CPU oracle for the D3M factorisation hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module, and
only as the checker / the timed CPU baseline.  The product package
``paper_2002_05018_b200`` never imports it; its CUDA path fails loudly when
the extension is missing.

What it is: a restatement of the reference's algorithm for the hot path
(``/root/reference/pkg/src/ddsolve``), with the five dense L1 kernels in C
(``d3m_oracle.c``, operation-for-operation identical to the numba JIT
backend, so pivots *and* values are bit-identical to the reference) and the
block-level drivers below in numpy (OpenBLAS ``@``, like the reference).

Pinning: ``tests/test_oracle_golden.py`` checks every function here against
the golden vectors in ``tests/golden/`` that ``tools/gen_golden.py`` produced by
running the reference itself in the build container, plus the reference's
own known-answer tests (``pkg/tests/test_dense_factor.py:16-31``,
``test_symbolic.py:32-39``, ``test_subdomain.py:133-143``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libd3m_oracle.so")
_SRC = os.path.join(_HERE, "d3m_oracle.c")

DEFAULT_PIVOT_TOL = 1e-12          # factor.py:19


def build(force: bool = False) -> str:
    """Compile the C restatement (gcc, no FMA contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        os.makedirs(os.path.dirname(_SO), exist_ok=True)
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math",
                               "-shared", "-fPIC", "-o", _SO, _SRC, "-lm"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        I = ctypes.c_int64
        D = ctypes.c_double
        _lib.d3m_oracle_bk_factor.restype = I
        _lib.d3m_oracle_bk_factor.argtypes = [P, I, I, D, P, P, P, P]
        _lib.d3m_oracle_bk_factor_m.restype = I
        _lib.d3m_oracle_bk_factor_m.argtypes = [P, I, I, D, P, P, P, P, P]
        for nm in ("d3m_oracle_solve_unit_lower", "d3m_oracle_solve_unit_lower_t"):
            getattr(_lib, nm).restype = None
            getattr(_lib, nm).argtypes = [P, I, I, P, I, I]
        for nm in ("d3m_oracle_apply_dinv_left", "d3m_oracle_apply_dinv_right"):
            getattr(_lib, nm).restype = None
            getattr(_lib, nm).argtypes = [P, P, P, I, P, I, I]
        _lib.d3m_oracle_hypot.restype = D
        _lib.d3m_oracle_hypot.argtypes = [D, D]
        _lib.d3m_oracle_bk_alpha.restype = D
        _lib.d3m_oracle_hypot_array.restype = None
        _lib.d3m_oracle_hypot_array.argtypes = [P, P, P, I]
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


# --------------------------------------------------------------------------
# L1 kernels (kernels.py:36-202), in-place like the reference.
# --------------------------------------------------------------------------

def bk_factor(W: np.ndarray, tol_abs: float, margin: np.ndarray | None = None):
    """kernels.py:36-146 -> (perm, tags, n2x2, growth, info); W in place.
    ``margin`` (2 doubles, optional) receives the pivot-decision margin and
    the argmax gap (the GPU kernels' diagnostic, include/d3m.h)."""
    assert W.dtype == np.complex128 and W.flags.c_contiguous
    n = W.shape[0]
    perm = np.empty(n, dtype=np.int64)
    tags = np.empty(n, dtype=np.int8)
    n2 = ctypes.c_int64(0)
    gr = ctypes.c_double(1.0)
    info = lib().d3m_oracle_bk_factor_m(_ptr(W), n, max(n, 1), float(tol_abs), _ptr(perm),
                                        _ptr(tags), ctypes.byref(n2), ctypes.byref(gr),
                                        _ptr(margin) if margin is not None else None)
    return perm, tags, int(n2.value), float(gr.value), int(info)


def bk_margins(M, pivot_tol=1e-12):
    """(decision margin, argmax gap) of the reference BK on M (a copy)."""
    W = np.array(M, dtype=np.complex128, order="C")
    mg = np.ones(2)
    bk_factor(W, pivot_tol * np.abs(W).max() if W.size else 0.0, mg)
    return float(mg[0]), float(mg[1])


def solve_unit_lower(L, B):
    """kernels.py:149-152, B (n x m, C order) in place."""
    n, m = B.shape
    lib().d3m_oracle_solve_unit_lower(_ptr(L), n, L.shape[1] if L.ndim == 2 else 1,
                                      _ptr(B), m, m)


def solve_unit_lower_t(L, B):
    """kernels.py:155-158."""
    n, m = B.shape
    lib().d3m_oracle_solve_unit_lower_t(_ptr(L), n, L.shape[1] if L.ndim == 2 else 1,
                                        _ptr(B), m, m)


def apply_dinv_left(d, e, tags, B):
    """kernels.py:161-181."""
    n, m = B.shape
    lib().d3m_oracle_apply_dinv_left(_ptr(d), _ptr(e), _ptr(tags), n, _ptr(B), m, m)


def apply_dinv_right(d, e, tags, B):
    """kernels.py:184-202."""
    rows, n = B.shape
    lib().d3m_oracle_apply_dinv_right(_ptr(d), _ptr(e), _ptr(tags), n, _ptr(B), rows, n)


def hypot(x: float, y: float) -> float:
    """glibc libm hypot (what numba's abs(complex) calls) -- NOT Python's
    math.hypot, which CPython implements with its own algorithm."""
    return lib().d3m_oracle_hypot(x, y)


def hypot_array(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    out = np.empty_like(x)
    lib().d3m_oracle_hypot_array(_ptr(x), _ptr(y), _ptr(out), x.size)
    return out


# --------------------------------------------------------------------------
# Dense factor (factor.py:30-116)
# --------------------------------------------------------------------------

class OracleSingular(Exception):
    pass


@dataclass
class OFactor:
    L: np.ndarray
    d: np.ndarray
    e: np.ndarray
    tags: np.ndarray
    perm: np.ndarray
    growth: float
    n_2x2: int
    info: int = -1
    scale: float = 0.0
    packed: np.ndarray | None = None     # the in-place W the kernel produced

    @property
    def n(self):
        return int(self.d.size)

    def solve(self, B):
        """factor.py:52-66."""
        one_d = np.ndim(B) == 1
        Z = np.array(B, dtype=np.complex128, ndmin=2)
        if one_d:
            Z = Z.T
        Z = np.ascontiguousarray(Z[self.perm, :])
        if self.n:
            solve_unit_lower(self.L, Z)
            apply_dinv_left(self.d, self.e, self.tags, Z)
            solve_unit_lower_t(self.L, Z)
        X = np.empty_like(Z)
        X[self.perm, :] = Z
        return X[:, 0] if one_d else X

    def dense_d(self):
        """factor.py:68-80."""
        D = np.diag(self.d).astype(np.complex128)
        for k in np.flatnonzero(self.tags == 2):
            D[k + 1, k] = D[k, k + 1] = self.e[k]
        return D


def dense_ldlt_bk(M, pivot_tol=DEFAULT_PIVOT_TOL, check_symmetry=True) -> OFactor:
    """factor.py:83-116 (errors raised as OracleSingular / ValueError)."""
    M = np.asarray(M)
    if M.ndim != 2 or M.shape[0] != M.shape[1]:
        raise ValueError("matrix must be square")
    n = M.shape[0]
    W = np.array(M, dtype=np.complex128, order="C")
    scale = float(np.abs(W).max()) if n else 0.0
    if check_symmetry and n and scale > 0.0:
        asym = np.abs(W - W.T).max()
        if asym > 1e-12 * scale:
            raise ValueError(f"matrix is not symmetric: max|M - M^T| = {asym:.3e}")
    perm, tags, n2, growth, info = bk_factor(W, pivot_tol * scale)
    if info >= 0:
        raise OracleSingular(f"no acceptable pivot at elimination step {info} "
                             f"(threshold {pivot_tol * scale:.3e})")
    packed = W.copy()
    L = np.tril(W, -1)
    d = np.diagonal(W).copy()
    e = np.zeros(n, dtype=np.complex128)
    two = np.flatnonzero(tags == 2)
    e[two] = W[two + 1, two]
    L[two + 1, two] = 0.0
    np.fill_diagonal(L, 1.0)
    return OFactor(L, d, e, tags, perm, growth, n2, info, scale, packed)


# --------------------------------------------------------------------------
# Host planning restated (symbolic.py:36-64, ordering.py:52-126,
# blockmat.py:123-129).  Graphs are lists of python sets.
# --------------------------------------------------------------------------

def clique_adjacency(nblocks, keys):
    adj = [set() for _ in range(nblocks)]
    for (i, j) in keys:
        if i != j:
            adj[i].add(j)
            adj[j].add(i)
    return adj


def _eliminate(adj_perm, n):
    """Elimination-graph pass in position order -> (pattern, parent)."""
    adj = [set(s) for s in adj_perm]
    pattern, parent = [], np.full(n, -1, dtype=np.int64)
    for j in range(n):
        rows = sorted(r for r in adj[j] if r > j)
        pattern.append(np.array(rows, dtype=np.int64))
        if rows:
            parent[j] = rows[0]
        for a in range(len(rows)):
            for b in range(a + 1, len(rows)):
                adj[rows[a]].add(rows[b])
                adj[rows[b]].add(rows[a])
    return pattern, parent


def symbolic_factor(adj, perm, sizes):
    """symbolic.py:36-64 -> dict(pattern, parent, sizes_perm, total)."""
    n = len(adj)
    perm = np.asarray(perm, dtype=np.int64)
    sizes = np.asarray(sizes, dtype=np.int64)
    inv = np.empty(n, dtype=np.int64)
    inv[perm] = np.arange(n)
    relab = [set() for _ in range(n)]
    for i in range(n):
        for j in adj[i]:
            relab[inv[i]].add(int(inv[j]))
    pattern, parent = _eliminate(relab, n)
    sp = sizes[perm]
    total = sum(int(sp[j]) * (int(sp[j]) + 1) // 2 + int(sp[j]) * int(sp[pattern[j]].sum())
                for j in range(n))
    return dict(pattern=pattern, parent=parent, sizes_perm=sp, total=total, perm=perm)


def min_degree_order(adj, weights):
    """ordering.py:52-79 (simplicial first, weighted degree, index)."""
    n = len(adj)
    adj = [set(s) for s in adj]
    alive = np.ones(n, dtype=bool)
    order = []
    for _ in range(n):
        best = None
        for v in np.flatnonzero(alive):
            nb = sorted(adj[v])
            simp = all(nb[b] in adj[nb[a]] for a in range(len(nb)) for b in range(a + 1, len(nb)))
            key = (0 if simp else 1, int(sum(int(weights[u]) for u in nb)), int(v))
            if best is None or key < best:
                best = key
        v = best[2]
        order.append(v)
        alive[v] = False
        nb = sorted(adj[v])
        for u in nb:
            adj[u].discard(v)
        for a in range(len(nb)):
            for b in range(a + 1, len(nb)):
                adj[nb[a]].add(nb[b])
                adj[nb[b]].add(nb[a])
    return np.array(order, dtype=np.int64)


def reorder(adj, weights):
    """ordering.py:105-126: keep min-degree only if not worse than natural."""
    n = len(adj)
    weights = np.asarray(weights, dtype=np.int64)
    md = min_degree_order(adj, weights)
    ident = np.arange(n, dtype=np.int64)
    if np.array_equal(md, ident):
        return md
    if symbolic_factor(adj, md, weights)["total"] <= symbolic_factor(adj, ident, weights)["total"]:
        return md
    return ident


# --------------------------------------------------------------------------
# Block LDL^T and block solve (factor.py:139-310)
# --------------------------------------------------------------------------

@dataclass
class OBlockFactor:
    plan: dict
    diag: list
    offdiag: dict
    stats: dict = field(default_factory=dict)


def permute_blocks(blocks, perm):
    """factor.py:139-151: relabel into elimination positions, lower storage."""
    n = len(perm)
    inv = np.empty(n, dtype=np.int64)
    inv[np.asarray(perm)] = np.arange(n)
    W = {}
    for (i, j), blk in blocks.items():
        a, b = int(inv[i]), int(inv[j])
        key, val = ((a, b), blk) if a >= b else ((b, a), blk.T)
        W[key] = W[key] + val if key in W else np.array(val, dtype=np.complex128, order="C")
    return W


def block_ldlt(blocks, plan, pivot_tol=DEFAULT_PIVOT_TOL, columns=None) -> OBlockFactor:
    """factor.py:154-240.  ``columns`` limits the elimination to the first
    block columns (used for the bounded CPU-baseline sample)."""
    sizes = plan["sizes_perm"]
    nb = len(sizes)
    W = permute_blocks(blocks, plan["perm"])
    diag, off = [], {}
    stored = 0
    flops = 0
    ncol = nb if columns is None else min(columns, nb)
    for j in range(ncol):
        nj = int(sizes[j])
        Kjj = W.pop((j, j), None)
        if Kjj is None:
            Kjj = np.zeros((nj, nj), dtype=np.complex128)
        try:
            fac = dense_ldlt_bk(Kjj, pivot_tol)
        except OracleSingular as err:
            raise OracleSingular(f"block column {j}: {err}") from err
        diag.append(fac)
        stored += nj * (nj + 1) // 2
        flops += nj ** 3 // 3 + nj ** 2
        rows = [int(r) for r in plan["pattern"][j]]
        X = {}
        for i in rows:
            ni = int(sizes[i])
            Kij = W.pop((i, j), None)
            if Kij is None:
                Kij = np.zeros((ni, nj), dtype=np.complex128)
            Y = np.ascontiguousarray(Kij[:, fac.perm].T)
            solve_unit_lower(fac.L, Y)
            X[i] = np.ascontiguousarray(Y.T)
            Lij = X[i].copy()
            apply_dinv_right(fac.d, fac.e, fac.tags, Lij)
            off[(i, j)] = Lij
            stored += ni * nj
            flops += ni * nj * nj + ni * nj
        for a, i in enumerate(rows):
            for kk in rows[:a + 1]:
                upd = X[i] @ off[(kk, j)].T
                flops += int(sizes[i]) * nj * int(sizes[kk])
                if i == kk:
                    upd = np.tril(upd) + np.tril(upd, -1).T
                W[(i, kk)] = W[(i, kk)] - upd if (i, kk) in W else -upd
    stats = dict(factor_entries=stored, flops=flops,
                 growth_factor=max((f.growth for f in diag), default=1.0),
                 n_2x2_pivots=sum(f.n_2x2 for f in diag))
    return OBlockFactor(plan, diag, off, stats)


def block_solve(F: OBlockFactor, g):
    """factor.py:243-310: one RHS column at a time, plan order."""
    plan = F.plan
    nb = len(plan["sizes_perm"])
    perm = plan["perm"]
    one_d = all(np.ndim(b) == 1 for b in g)
    blocks = [np.array(b, dtype=np.complex128, ndmin=2).T if np.ndim(b) == 1
              else np.array(b, dtype=np.complex128) for b in g]
    cols = blocks[0].shape[1] if nb else 0
    out = [np.empty((b.shape[0], cols), dtype=np.complex128) for b in blocks]
    pattern = plan["pattern"]
    for c in range(cols):
        b = [blocks[int(perm[j])][:, c:c + 1].copy() for j in range(nb)]
        u = []
        for j in range(nb):
            fac = F.diag[j]
            z = np.ascontiguousarray(b[j][fac.perm, :])
            solve_unit_lower(fac.L, z)
            for i in pattern[j]:
                b[int(i)] = b[int(i)] - F.offdiag[(int(i), j)] @ z
            u.append(z)
        for j in range(nb):
            apply_dinv_left(F.diag[j].d, F.diag[j].e, F.diag[j].tags, u[j])
        x = [None] * nb
        for j in range(nb - 1, -1, -1):
            fac = F.diag[j]
            w = u[j]
            for i in pattern[j]:
                w = w - F.offdiag[(int(i), j)].T @ x[int(i)]
            w = np.ascontiguousarray(w)
            solve_unit_lower_t(fac.L, w)
            xj = np.empty_like(w)
            xj[fac.perm, :] = w
            x[j] = xj
        for j in range(nb):
            out[int(perm[j])][:, c:c + 1] = x[j]
    return [o[:, 0] for o in out] if one_d else out


# --------------------------------------------------------------------------
# DDM layer (subdomain.py:166-237)
# --------------------------------------------------------------------------

def reduce_domain(A, D_all, f, pivot_tol=DEFAULT_PIVOT_TOL):
    """subdomain.py:166-184 -> (K_D, g_d, factor)."""
    fac = dense_ldlt_bk(A, pivot_tol)
    rhs = np.concatenate([D_all, np.asarray(f)[:, None]], axis=1)
    X = fac.solve(rhs)
    K = D_all.T @ X[:, :-1]
    K = 0.5 * (K + K.T)
    g = D_all.T @ X[:, -1]
    return K, g, fac


def assemble_reduced(reduced, incident, sizes):
    """subdomain.py:187-214 with blockmat.add_block (blockmat.py:69-81):
    ``incident[d]`` lists domain d's interfaces in coupling order."""
    sizes = np.asarray(sizes, dtype=np.int64)
    blocks = {}
    g = [np.zeros(int(s), dtype=np.complex128) for s in sizes]
    for d, (K_D, g_d) in enumerate(reduced):
        ifs = list(incident[d])
        off = np.concatenate([[0], np.cumsum(sizes[ifs])]).astype(np.int64)
        for a, ia in enumerate(ifs):
            g[ia] = g[ia] + g_d[off[a]:off[a + 1]]
            for b, ib in enumerate(ifs):
                if ia < ib:
                    continue
                sub = np.asarray(K_D[off[a]:off[a + 1], off[b]:off[b + 1]], dtype=np.complex128)
                blocks[(ia, ib)] = blocks[(ia, ib)] + sub if (ia, ib) in blocks else sub.copy()
    return blocks, g


def recover_primal(factors, f_list, couplings, dof_maps, lam):
    """subdomain.py:217-237: E_d = A_d^-1 (f_d - sum_c D_c lam_c), averaged."""
    n_glob = 1 + max(int(np.max(m)) for m in dof_maps)
    acc = np.zeros(n_glob, dtype=np.complex128)
    cnt = np.zeros(n_glob)
    for fac, f, cps, dm in zip(factors, f_list, couplings, dof_maps):
        rhs = np.array(f, dtype=np.complex128)
        for (itf, D) in cps:
            if D.shape[1]:
                rhs = rhs - D @ lam[itf]
        E = fac.solve(rhs)
        acc[dm] += E
        cnt[dm] += 1.0
    return acc / cnt

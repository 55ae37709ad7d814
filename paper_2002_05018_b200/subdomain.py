"""DDM layer of the hot path on the GPU: Schur reduction of the subdomains,
assembly of the block-sparse interface matrix, primal recovery.

Drop-in for subdomain.py (pkg/src/ddsolve/subdomain.py:34-237): same
dataclasses, names, errors and messages.  ``reduce_domains`` is the batched
entry point (all subdomains of equal shape in flight in one launch chain);
``reduce_domain`` keeps the reference's one-domain signature.  Results stay in
HBM (``DeviceArray``) so assembly, factorisation, solve and recovery chain
without host round trips.

The finite-element front end (build_subdomain_systems, the 2-D mesh) is out
of scope for this hot-path build.
"""

from __future__ import annotations

import zlib
from dataclasses import dataclass, field

import os

import numpy as np

from . import _lib
from .blockmat import BlockSparseSym
from .device import BatchHost, DeviceArray, empty, require_cuda, stream_ptr, to_device, upload_bytes, upload_i64
from .factor import DEFAULT_PIVOT_TOL, DenseFactor, SolverStateError, _collect, _singular_msg

_P = _lib.ptr


class SingularDomainError(Exception):
    pass


@dataclass
class Coupling:
    interface: int
    D: np.ndarray          # local dofs x kept multiplier dofs
    sign: int


@dataclass
class SubdomainSystem:
    domain: int
    A: np.ndarray
    f: np.ndarray
    dof_map: np.ndarray
    couplings: list = field(default_factory=list)
    factor: DenseFactor | None = None

    @property
    def n_dofs(self) -> int:
        return int(np.asarray(self.dof_map).size)


@dataclass
class ReducedSystem:
    K: BlockSparseSym
    g: list
    interface_sizes: np.ndarray
    lam: list | None = None

    @property
    def n_lambda(self) -> int:
        return int(np.asarray(self.interface_sizes).sum())


def interface_lambda_nodes(part) -> list[np.ndarray]:
    """Kept multiplier dofs per interface (subdomain.py:75-111): at a node
    shared by several interfaces, scanned in ascending interface order, an
    interface whose (dom_lo, dom_hi) pair closes a cycle among the domains
    already connected there drops its dof."""
    at_node: dict[int, list[int]] = {}
    for k, itf in enumerate(part.interfaces):
        for v in itf.nodes:
            at_node.setdefault(int(v), []).append(k)
    dropped = set()
    for v in sorted(at_node):
        ifs = sorted(at_node[v])
        if len(ifs) < 2:
            continue
        root: dict[int, int] = {}

        def find(x):
            root.setdefault(x, x)
            while root[x] != x:
                root[x] = root[root[x]]
                x = root[x]
            return x

        for k in ifs:
            ra, rb = find(part.interfaces[k].dom_lo), find(part.interfaces[k].dom_hi)
            if ra == rb:
                dropped.add((k, v))
            else:
                root[ra] = rb
    return [np.array([int(v) for v in itf.nodes if (k, int(v)) not in dropped], dtype=np.int64)
            for k, itf in enumerate(part.interfaces)]


_FP_MAX_BYTES = 256 << 20


def _fingerprint(a):
    """CRC-32 of a host array's bytes (numpy, CPU tensor or SparseBlock), or
    None for device arrays and arrays above _FP_MAX_BYTES.  recover_primal
    reuses X = A^-1 [D | F] only while the loads it was formed from are the
    same objects with the same content (an in-place edit of f, e.g. a new
    excitation, is seen) and the couplings are the same objects.  Couplings
    are not content-hashed: they are geometry (config 5 carries 1.9 GB of
    them, ~0.4 s of CRC per call) and must not be edited in place after
    reduce_domains -- reduce again instead."""
    if isinstance(a, SparseBlock):
        if a.keys.nbytes + a.vals.nbytes > _FP_MAX_BYTES:
            return None
        return (zlib.crc32(a.keys.view(np.uint8)), zlib.crc32(a.vals.view(np.uint8)))
    if isinstance(a, DeviceArray) or (type(a).__module__.startswith("torch") and a.is_cuda):
        return None
    arr = a.numpy() if type(a).__module__.startswith("torch") else np.asarray(a)
    if arr.nbytes > _FP_MAX_BYTES:
        return None
    return zlib.crc32(np.ascontiguousarray(arr).view(np.uint8))


class SparseBlock:
    """A dense subdomain block (A_d or D_d) carried as unique-key COO.

    FEM subdomain matrices have ~30 nonzeros per row, so shipping the dense
    n x n array costs ~n/30 times more host->device traffic than the entries.
    ``keys`` are row-major positions r * ncols + c (unique, ascending), and
    ``vals`` the exact dense values at those positions (every other entry is
    +0.0); ``np.asarray`` gives the dense array of the reference API
    (subdomain.py:124-163 builds dense A_d / D_d), and reduce_domains
    densifies on the device with one scatter, bit-identical to uploading the
    dense array."""

    ndim = 2
    dtype = np.dtype(np.complex128)

    def __init__(self, shape, keys, vals):
        self.shape = (int(shape[0]), int(shape[1]))
        self.keys = np.ascontiguousarray(keys, dtype=np.int64)
        self.vals = np.ascontiguousarray(vals, dtype=np.complex128)

    def pinned(self, t):
        """(keys, vals) as torch CPU tensors in page-locked memory.  The first
        upload moves the entries there once and turns ``keys`` / ``vals`` into
        views of it, so later edits of the arrays are seen and every upload is
        a direct DMA (from pageable memory the copies of config 2's eight
        blocks cost ~5 ms per reduction)."""
        if getattr(self, "_pin", None) is None:
            pk = t.from_numpy(self.keys).pin_memory()
            pv = t.from_numpy(self.vals).pin_memory()
            self.keys, self.vals = pk.numpy(), pv.numpy()
            self._pin = (pk, pv)
        return self._pin

    def toarray(self) -> np.ndarray:
        out = np.zeros(self.shape, dtype=np.complex128)
        out.reshape(-1)[self.keys] = self.vals
        return out

    def __array__(self, dtype=None, copy=None):
        a = self.toarray()
        return a if dtype is None else a.astype(dtype)

    @property
    def T(self) -> np.ndarray:
        return self.toarray().T

    @staticmethod
    def hconcat(blocks, sort: bool = True) -> "SparseBlock":
        """[D_1 | D_2 | ...] as one block.  ``sort=False`` skips the key sort
        (the argsort is most of the cost, ~1.5 ms per config-2 domain): enough
        for a device scatter, which takes the entries in any order."""
        n = blocks[0].shape[0]
        m = sum(b.shape[1] for b in blocks)
        keys, vals, off = [], [], 0
        for b in blocks:
            r, c = np.divmod(b.keys, max(b.shape[1], 1))
            keys.append(r * m + off + c)
            vals.append(b.vals)
            off += b.shape[1]
        k = np.concatenate(keys) if keys else np.zeros(0, np.int64)
        v = np.concatenate(vals) if vals else np.zeros(0, np.complex128)
        if sort:
            o = np.argsort(k, kind="stable")
            k, v = k[o], v[o]
        out = SparseBlock((n, m), k, v)
        out._transient = True          # built per call: not worth page-locking
        return out


def _coupling_matrix(sys: SubdomainSystem, sort: bool = True):
    if sys.couplings and all(isinstance(c.D, SparseBlock) for c in sys.couplings):
        return SparseBlock.hconcat([c.D for c in sys.couplings], sort=sort)
    if sys.couplings:
        return np.concatenate([np.asarray(c.D, dtype=np.complex128) for c in sys.couplings], axis=1)
    return np.zeros((sys.n_dofs, 0), dtype=np.complex128)


def _load_cols(s) -> int:
    shp = tuple(s.f.shape) if hasattr(s.f, "shape") else np.shape(s.f)
    return 1 if len(shp) == 1 else int(shp[1])


def _domain_bytes(n: int, m: int, r: int) -> int:
    """Device bytes one domain of a reduce batch holds (A, D, F, X, Z, C, K, G,
    panel workspace)."""
    w = m + r
    # A, D, F, X, Z, C, K, G, the compact D rows of D^T X (<= 0.6 n), panel workspace
    return 16 * (n * n + n * m + n * r + 2 * n * w + m * w + m * m + m * r + (6 * n * m) // 10) + 129 * 16 * n + 1024


def _free_bytes(t) -> int:
    free, _ = t.cuda.mem_get_info()
    return int(free + t.cuda.memory_reserved() - t.cuda.memory_allocated())


def reduce_domains(systems: list[SubdomainSystem], pivot_tol: float = DEFAULT_PIVOT_TOL, keep: str = "factor",
                   max_batch_bytes: int | None = None, margins: bool = False) -> list:
    """Batched reduce_domain (subdomain.py:166-184): subdomains of equal order n
    are factored and reduced together (BK -> multi-RHS solve -> D^T X on DMMA
    -> symmetrisation), in batches sized to the free device memory (or
    ``max_batch_bytes``).  Returns [(K_D, g_d)] as DeviceArrays; g_d is m x r
    when the systems carry r load columns (f of shape n x r), else a vector.

    keep="factor" caches each DenseFactor on its system, like the reference.
    keep="solution" keeps X_d = A_d^-1 [D_d | F_d] (n x (m + r)) instead and
    releases the factor values, so recover_primal forms
    E_d = X_F - X_D lambda_d with one GEMM (exact-arithmetic equal to the
    reference's A_d^-1 (F_d - D_d lambda_d)); it is what lets config 5
    (64 x n = 13,428, 185 GB of factors) run in 180 GB of HBM.  keep="auto"
    chooses "solution" when all factors would not fit in half the free
    device memory.  keep="schur" keeps the factor but forms only the Schur
    blocks, as K = Z_D^T D^-1 Z with Z = L^-1 P [D | F] (A^-1 = P^T L^-T D^-1
    L^-1 P): no backward sweep, no X (recover_primal then solves with the
    factor) -- for reductions whose primal recovery is not needed (config 3).

    ``margins`` tracks each subdomain factorisation's pivot-decision margins
    (DenseFactor.margin; include/d3m.h d3m_bk_factor_batched)."""
    t = require_cuda()
    if keep not in ("factor", "solution", "auto", "schur"):
        raise ValueError(f"keep must be 'factor', 'solution', 'auto' or 'schur', not {keep!r}")
    # one batch per subdomain order n (the factorisation does not depend on
    # m); coupling blocks are zero-padded to the group's largest m and each
    # domain's K_D / g_d is the leading m x m / m view of its padded result
    groups: dict[int, list[int]] = {}
    ms = []
    for idx, s in enumerate(systems):
        n = int(np.shape(s.A)[0]) if not isinstance(s.A, DeviceArray) else s.A.shape[0]
        ms.append(sum(int(np.shape(c.D)[1]) for c in s.couplings))
        groups.setdefault(n, []).append(idx)
    rs = {_load_cols(s) for s in systems}
    if len(rs) > 1:
        raise ValueError("all subdomains must carry the same number of load columns")
    r = rs.pop() if rs else 1
    vec = bool(systems) and len(np.shape(systems[0].f) if not hasattr(systems[0].f, "shape")
                                else tuple(systems[0].f.shape)) == 1
    if keep == "auto":
        fac = sum(16 * n * n * len(mem) for n, mem in groups.items())
        keep = "solution" if fac > 0.5 * _free_bytes(t) else "factor"
    out = [None] * len(systems)
    first_error = None
    for n, members in groups.items():
        # largest coupling first, so each memory-sized batch pads to a close m
        members = sorted(members, key=lambda i: -ms[i])
        pos = 0
        while pos < len(members):
            m = ms[members[pos]]
            budget = max_batch_bytes if max_batch_bytes is not None else int(0.8 * _free_bytes(t))
            # the split upload of dense host matrices keeps an intact copy A0
            per = _domain_bytes(n, m, r) + (16 * n * n if n > _lib.PANEL_BK_MIN and _host_dense(systems[members[pos]].A)
                                            else 0)
            cap = max(1, budget // per)
            chunk = members[pos:pos + cap]
            pos += len(chunk)
            err = _reduce_chunk(systems, chunk, n, m, r, ms, pivot_tol, keep, vec, out, margins)
            if err is not None and (first_error is None or err[0] < first_error[0]):
                first_error = err
    if first_error is not None:
        raise first_error[1]
    return out


def _host_dense(a) -> bool:
    """A dense host matrix (numpy array or CPU torch tensor)."""
    if isinstance(a, (SparseBlock, DeviceArray)):
        return False
    if type(a).__module__.startswith("torch"):
        return not a.is_cuda
    return isinstance(a, np.ndarray)


_COPY_STREAMS: dict = {}


def _copy_stream(t):
    dev = t.cuda.current_device()
    if dev not in _COPY_STREAMS:
        _COPY_STREAMS[dev] = t.cuda.Stream()
    return _COPY_STREAMS[dev]


def _host_matrix_ptrs(systems, members, n):
    """Contiguous complex128 host views of the members' A and a ctypes array
    of their data pointers (the views are returned so they outlive the copies)."""
    t = require_cuda()
    views, ptrs = [], []
    for idx in members:
        a = systems[idx].A
        if type(a).__module__.startswith("torch"):
            a = a.to(dtype=t.complex128).contiguous()
            p = a.data_ptr()
        else:
            a = np.ascontiguousarray(np.asarray(a, dtype=np.complex128))
            p = a.ctypes.data
        if tuple(a.shape) != (n, n):
            raise ValueError(f"domain {systems[idx].domain}: A must be {n} x {n}")
        views.append(a)
        ptrs.append(p)
    return views, (_lib.ctypes.c_void_p * len(ptrs))(*ptrs)


def _fill_inputs(systems, members, n, ms, A, D, f):
    for i, idx in enumerate(members):
        s = systems[idx]
        mr = ms[idx]
        if A is not None:
            _fill(A[i], s.A, (n, n))
        if mr:
            if _dev_D(s):
                D[i, :, :mr].copy_(s._d3m_D)
            elif len(s.couplings) == 1:
                _fill(D[i, :, :mr], s.couplings[0].D, (n, mr))
            elif all(isinstance(c.D, SparseBlock) for c in s.couplings):
                # each interface's block straight into its column range (page-locked entries, no host
                # concatenation: that cost ~1.8 ms per config-2 domain)
                off = 0
                for c in s.couplings:
                    mc = int(c.D.shape[1])
                    _fill(D[i, :, off:off + mc], c.D, (n, mc))
                    off += mc
            else:
                _fill(D[i, :, :mr], _coupling_matrix(s, sort=False), (n, mr))
        _fill(f[i], s.f, (n, f.shape[2]))


def _reduce_chunk(systems, members, n, m, r, ms, pivot_tol, keep, vec, out, margins=False, A_dev=None):
    """One batch of equal-order subdomains through d3m_schur_reduce_batched.

    Dense host matrices on the panel-BK path (n > 512) take the split upload:
    the lower row blocks of every A_d go first (d3m_copy_triangle part 0, on
    the compute stream) and are duplicated device-side into an intact copy
    A0; the panel BK starts on them at once (it reads nothing else: scale
    over the lower triangle, d3m_bk_panel_batched check_sym bit 3) while a
    copy stream uploads D, F and the upper remainder into A0 and runs the
    symmetry check and full scale there (d3m_sym_scan_batched,
    factor.py:94-98).  An input whose full scale differs from the lower
    triangle's, or that fails the check, is reduced again from A0 by the
    one-pass path, which applies the reference's check and threshold
    exactly.  ``A_dev``: device matrices already in place (that re-run)."""
    t = require_cuda()
    B = len(members)
    split = A_dev is None and n > _lib.PANEL_BK_MIN and all(_host_dense(systems[i].A) for i in members)
    A = empty((B, n, n)) if A_dev is None else A_dev
    D = t.zeros((B, n, m), dtype=t.complex128, device="cuda")
    f = empty((B, n, r))
    perm = t.empty((B, n), dtype=t.int64, device="cuda")
    tags = t.empty((B, n), dtype=t.int8, device="cuda")
    n2 = t.empty(B, dtype=t.int32, device="cuda")
    info = t.empty(B, dtype=t.int32, device="cuda")
    gr = t.empty(B, dtype=t.float64, device="cuda")
    sc = t.empty(B, dtype=t.float64, device="cuda")
    asy = t.empty(B, dtype=t.float64, device="cuda")
    K = empty((B, m, m))
    g = empty((B, m, r))
    wz = empty((B, n, m + r))
    wx = empty((B, n, m + r))
    wc = empty((B, max(m, 1), m + r))
    if n > _lib.PANEL_BK_MIN:
        nbytes = int(_lib.load().d3m_bk_panel_workspace(n, B))
        scratch = t.empty((nbytes + 15) // 16, dtype=t.complex128, device="cuda")
        d_tasks = t.empty(64 * max(B, 4 * ((n + 63) // 64) * B), dtype=t.uint8, device="cuda")
    else:
        scratch = empty((B, 4 * n)) if 64 * n > 200 * 1024 else None
        d_tasks = t.empty(64 * B, dtype=t.uint8, device="cuda")
    mg = t.empty((B, 2), dtype=t.float64, device="cuda") if margins else None
    flags = 1 if keep == "schur" else 0
    if split:
        S, cs = t.cuda.current_stream(), _copy_stream(t)
        views, hptr = _host_matrix_ptrs(systems, members, n)
        _lib.call("d3m_copy_triangle", B, hptr, n, _P(A), n * n, n, n, 0, 1, stream_ptr())
        A0 = A.clone()             # one flat D2D copy (the upper halves are overwritten below)
        cs.wait_event(S.record_event())
        _lib.call("d3m_bk_panel_batched", B, n, _P(A), n * n, n, float(pivot_tol), 8, _P(perm), _P(tags), _P(n2),
                  _P(gr), _P(info), _P(sc), _P(asy), _P(scratch), _P(mg), stream_ptr())
        flags |= 2
        sc_full = t.empty(B, dtype=t.float64, device="cuda")
        asy_full = t.empty(B, dtype=t.float64, device="cuda")
        red = t.empty(8 * B, dtype=t.float64, device="cuda")
        with t.cuda.stream(cs):
            _fill_inputs(systems, members, n, ms, None, D, f)
            ev_df = cs.record_event()
            cstream = _lib.ctypes.c_void_p(cs.cuda_stream)
            _lib.call("d3m_copy_triangle", B, hptr, n, _P(A0), n * n, n, n, 1, 1, cstream)
            _lib.call("d3m_sym_scan_batched", B, n, _P(A0), n * n, n, _P(sc_full), _P(asy_full), _P(red), cstream)
            ev_scan = cs.record_event()
        S.wait_event(ev_df)
    else:
        _fill_inputs(systems, members, n, ms, A if A_dev is None else None, D, f)
    rows, nrows = _nonzero_rows(D, n) if keep != "schur" else (None, 0)
    wd = empty((B, nrows, m)) if rows is not None else None
    # the coupling columns each domain really has (its D is zero-padded to the batch's m): the blocked
    # solves skip the padded ones
    mcols = np.array([ms[i] for i in members], dtype=np.int32)
    _lib.call("d3m_schur_reduce_batched", B, n, m, r, _P(A), _P(D), _P(f), float(pivot_tol), _P(perm),
              _P(tags), _P(n2), _P(gr), _P(info), _P(sc), _P(asy), _P(K), _P(g), _P(wz), _P(wx), _P(wc),
              _P(scratch), _P(d_tasks), _P(rows), int(nrows), _P(wd), flags, _P(mg),
              _lib.hptr(mcols) if bool(np.any(mcols < m)) else None, stream_ptr())
    if split:
        S.wait_event(ev_scan)
        sc_h, full_h, asy_h = sc.cpu().numpy(), sc_full.cpu().numpy(), asy_full.cpu().numpy()
        del views
        if not np.array_equal(sc_h, full_h) or bool(np.any(asy_h > 1e-12 * full_h)):
            del A, D, f, wz, wx, wc, K, g, scratch, wd, rows
            return _reduce_chunk(systems, members, n, m, r, ms, pivot_tol, keep, vec, out, margins, A_dev=A0)
        asy.copy_(asy_full)
        # the reference leaves the input's upper triangle in `packed`
        # (kernels.py:18): bring it over from the intact copy (device to device)
        dptr = (_lib.ctypes.c_void_p * B)(*[A0.data_ptr() + 16 * n * n * b for b in range(B)])
        _lib.call("d3m_copy_triangle", B, dptr, n, _P(A), n * n, n, n, 1, 3, stream_ptr())
        del A0
    del wd, rows
    del wz, scratch, wc
    try:
        facs = _collect(A, perm, tags, n2, info, gr, sc, asy, pivot_tol, None,
                        wrap=lambda b, msg: SingularDomainError(
                            f"domain {systems[members[b]].domain} is singular: {msg}"), margin=mg)
    except (SingularDomainError, ValueError) as err:
        return (members[int(_first_bad(info))], err)
    kh, gh = BatchHost(K), BatchHost(g)
    for i, idx in enumerate(members):
        s = systems[idx]
        mr = ms[idx]
        # X = A^-1 [D | F] (m padded) is kept in both modes: recover_primal
        # forms E = X_F - X_D lambda from it while the loads and couplings are
        # the arrays reduced here (identity check), else solves with the factor
        if keep == "schur":            # no X: recovery solves with the factor
            s._d3m_X, s._d3m_src = None, None
        else:
            s._d3m_X = wx[i]
            s._d3m_Xm = m
            s._d3m_src = (s.f, tuple(c.D for c in s.couplings), _fingerprint(s.f))
        if keep in ("factor", "schur"):
            s.factor = facs[i]
            s._d3m_D = D[i, :, :mr]
        else:
            s.factor = facs[i].release()
            s._d3m_D = None
        gidx = (i, slice(0, mr), 0) if vec else (i, slice(0, mr), slice(None))
        out[idx] = (DeviceArray(K[i, :mr, :mr], (kh, (i, slice(0, mr), slice(0, mr)))),
                    DeviceArray(g[gidx], (gh, gidx)))
    return None


def _nonzero_rows(D, n):
    """Rows where each domain's coupling block D_d (the filled device batch
    B x n x m) has nonzeros, ascending and -1 padded to the batch maximum,
    for D^T X over those rows only; (None, 0) when the couplings are dense
    enough that the full product is as cheap.  One device pass over D
    (d3m_nonzero_rows), one sync for the counts."""
    t = require_cuda()
    B, m = int(D.shape[0]), int(D.shape[2])
    if m == 0 or n == 0 or B == 0:
        return None, 0
    flag = t.empty(B * n, dtype=t.int8, device="cuda")
    idx = t.empty((B, n), dtype=t.int64, device="cuda")
    cnt = t.empty(B, dtype=t.int32, device="cuda")
    _lib.call("d3m_nonzero_rows", B, n, m, _P(D), _P(flag), _P(idx), _P(cnt), stream_ptr())
    nrows = int(cnt.cpu().numpy().max())
    if nrows == 0 or nrows > 0.6 * n:
        return None, 0
    return idx[:, :nrows].contiguous(), nrows


def _fill(dst, src, shape):
    """Copy a host array or device handle into a device slice (one H2D copy
    straight from the numpy buffer for host inputs)."""
    t = require_cuda()
    if isinstance(src, SparseBlock):
        assert tuple(src.shape) == tuple(shape)
        dst.zero_()
        if src.keys.size:
            if getattr(src, "_transient", False):
                k = t.from_numpy(src.keys).to("cuda", non_blocking=False)
                v = t.from_numpy(src.vals).to("cuda", non_blocking=False)
            else:
                hk, hv = src.pinned(t)
                k = hk.to("cuda", non_blocking=True)
                v = hv.to("cuda", non_blocking=True)
            if dst.is_contiguous():
                dst.view(-1).index_put_((k,), v)
            else:
                dst[k // shape[1], k % shape[1]] = v
        return
    if type(src).__module__.startswith("torch") and not src.is_cuda:      # host tensor (pinned: async DMA)
        dst.copy_(src.reshape(shape), non_blocking=bool(src.is_pinned()))
    elif isinstance(src, DeviceArray) or type(src).__module__.startswith("torch"):
        dst.copy_(to_device(src).reshape(shape))
    else:
        dst.copy_(t.from_numpy(np.ascontiguousarray(np.asarray(src, dtype=np.complex128)).reshape(shape)))


def _dev_D(s) -> bool:
    return getattr(s, "_d3m_D", None) is not None


def _first_bad(info) -> int:
    h = info.cpu().numpy()
    return int(np.flatnonzero(h != -1)[0])


def reduce_domain(sys: SubdomainSystem, pivot_tol: float = DEFAULT_PIVOT_TOL):
    """K_D = D^T A^-1 D (symmetrised) and g_d = D^T A^-1 f for one domain
    (subdomain.py:166-184); the factor is cached on ``sys``."""
    return reduce_domains([sys], pivot_tol)[0]


def assemble_reduced(reduced, part) -> ReducedSystem:
    """Scatter per-domain Schur blocks into the block-sparse reduced system
    (subdomain.py:187-214).  ``reduced[d]`` is ordered by
    ``part.incident_interfaces(d)``.  Block (ia, ib) = sum over domains in
    ascending order (first contribution copied, later ones added, like
    blockmat.add_block), done on the device when the inputs are resident."""
    lam_nodes = interface_lambda_nodes(part)
    sizes = np.array([ln.size for ln in lam_nodes], dtype=np.int64)
    contrib: dict[tuple[int, int], list] = {}
    gcontrib: dict[int, list] = {}
    device = True
    for d, (K_D, g_d) in enumerate(reduced):
        ifaces = [int(i) for i in part.incident_interfaces(d)]
        off = np.concatenate([[0], np.cumsum(sizes[ifaces])]).astype(np.int64)
        if tuple(K_D.shape) != (int(off[-1]), int(off[-1])):
            raise ValueError(f"domain {d}: reduced block is {tuple(K_D.shape)}, expected "
                             f"({int(off[-1])}, {int(off[-1])})")
        device &= isinstance(K_D, DeviceArray) and isinstance(g_d, DeviceArray)
        for a, ia in enumerate(ifaces):
            gcontrib.setdefault(ia, []).append((g_d, int(off[a]), int(sizes[ia])))
            for b, ib in enumerate(ifaces):
                if ia >= ib:
                    contrib.setdefault((ia, ib), []).append((K_D, int(off[a]), int(off[b])))
    if not device:
        return _assemble_host(contrib, gcontrib, sizes)
    return _assemble_device(contrib, gcontrib, sizes)


def _assemble_host(contrib, gcontrib, sizes):
    K = BlockSparseSym(sizes)
    for (ia, ib), lst in contrib.items():
        for (KD, oa, ob) in lst:
            KDh = np.asarray(KD)
            K.add_block(ia, ib, KDh[oa:oa + sizes[ia], ob:ob + sizes[ib]])
    K.validate()
    cols = {np.asarray(gd).shape[1:] for lst in gcontrib.values() for (gd, _, _) in lst}
    tail = cols.pop() if len(cols) == 1 else ()
    g = [np.zeros((int(s),) + tuple(tail), dtype=np.complex128) for s in sizes]
    for ia, lst in gcontrib.items():
        for (gd, o, n) in lst:
            g[ia] = g[ia] + np.asarray(gd)[o:o + n]
    return ReducedSystem(K, g, sizes)


def _assemble_device(contrib, gcontrib, sizes):
    t = require_cuda()
    keys = list(contrib)
    koff, tot = {}, 0
    for key in keys:
        koff[key] = tot
        tot += int(sizes[key[0]]) * int(sizes[key[1]])
    goff = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    gcols = {tuple(gd.shape[1:]) for lst in gcontrib.values() for (gd, _, _) in lst}
    if len(gcols) > 1:
        raise ValueError("reduced loads carry different numbers of columns")
    gtail = gcols.pop() if gcols else ()
    rg = int(gtail[0]) if gtail else 1
    kpool = empty(max(tot, 1))
    gpool = t.zeros(max(int(goff[-1]) * rg, 1), dtype=t.complex128, device="cuda")
    rounds: dict[tuple[int, int], list] = {}     # (round, base) -> tasks

    def src_of(dev: DeviceArray):
        st = dev.tensor
        base = st.untyped_storage().data_ptr()
        return base, st, (st.data_ptr() - base) // 16

    bases = {}
    for key, lst in contrib.items():
        ia, ib = key
        for r, (KD, oa, ob) in enumerate(lst):
            base, st, o = src_of(KD)
            bases[base] = st
            ld = int(KD.tensor.stride(0))
            rounds.setdefault((r, base, "K"), []).append(
                (o + oa * ld + ob, koff[key], int(sizes[ia]), int(sizes[ib]), ld, int(sizes[ib]), 0,
                 _lib.COPY_STORE if r == 0 else _lib.COPY_ADD))
    for ia, lst in gcontrib.items():
        for r, (gd, o0, n) in enumerate(lst):
            base, st, o = src_of(gd)
            bases[base] = st
            mode = _lib.COPY_ZERO_ADD if r == 0 else _lib.COPY_ADD
            if not gtail:
                rec = (o + o0, int(goff[ia]), 1, n, n, n, 0, mode)
            else:               # g_d is m x rg with row stride ld
                ld = int(gd.tensor.stride(0))
                rec = (o + o0 * ld, int(goff[ia]) * rg, n, rg, ld, rg, 0, mode)
            rounds.setdefault((r, base, "g"), []).append(rec)
    for (r, base, what) in sorted(rounds, key=lambda x: (x[0], x[2], x[1])):
        recs = np.array(rounds[(r, base, what)], dtype=_lib.COPY_TASK)
        st = bases[base]
        whole = t.empty(0, dtype=t.complex128, device="cuda").set_(
            st.untyped_storage(), 0, (st.untyped_storage().nbytes() // 16,))
        dst = kpool if what == "K" else gpool
        maxe = int((recs["rows"].astype(np.int64) * recs["cols"]).max())
        d_recs = upload_bytes(recs)          # keep alive until the launch is enqueued
        _lib.call("d3m_block_copy", _P(whole), _P(dst), _P(d_recs), len(recs), maxe, stream_ptr())
    K = BlockSparseSym(sizes)
    for key in keys:
        o, ni, nj = koff[key], int(sizes[key[0]]), int(sizes[key[1]])
        K.blocks[key] = DeviceArray(kpool[o:o + ni * nj].reshape(ni, nj))
    K._d3m_pool = kpool
    if gtail:
        g = [DeviceArray(gpool[int(goff[i]) * rg:int(goff[i + 1]) * rg].reshape(int(sizes[i]), rg))
             for i in range(sizes.size)]
    else:
        g = [DeviceArray(gpool[int(goff[i]):int(goff[i + 1])]) for i in range(sizes.size)]
    return ReducedSystem(K, g, sizes)


def _as_batch(views, shape):
    """Stack equally shaped device views without a copy when they already sit
    at a constant stride in one allocation (a reduce batch), else stack."""
    t = require_cuda()
    v0 = views[0]
    numel = int(np.prod(shape))
    if all(v.is_contiguous() for v in views) and \
            all(v.untyped_storage().data_ptr() == v0.untyped_storage().data_ptr() for v in views):
        step = (views[1].data_ptr() - v0.data_ptr()) // v0.element_size() if len(views) > 1 else numel
        if step >= numel and all(views[i].data_ptr() - v0.data_ptr() == i * step * v0.element_size()
                                 for i in range(len(views))):
            return v0.as_strided((len(views),) + tuple(shape), (step,) + tuple(v0.stride())), step
    return t.stack([v.reshape(shape) for v in views]).contiguous(), numel


def recover_primal(systems: list[SubdomainSystem], lam: list) -> np.ndarray | DeviceArray:
    """E_d = A_d^-1 (f_d - D_d lambda) with the cached factors, assembled
    with averaging of duplicated interface dofs (subdomain.py:217-237).
    Multi-column loads (lambda_i of shape size_i x r) give E of shape
    n_glob x r.  While the loads and couplings are the arrays reduce_domains
    saw, E_d = X_F - X_D lambda_d is formed from the retained
    X_d = A_d^-1 [D_d | F_d] with one GEMM (exact-arithmetic equal; tests
    compare it with the factor solve to 1e-9); otherwise the cached factor
    solves A_d^-1 (f_d - D_d lambda_d) as the reference does."""
    ET, e_off, r, one_d = _local_E(systems, lam)
    outT = _ordered_average(systems, ET, e_off, r)
    out = outT[0] if one_d else outT.t().contiguous()
    if all(isinstance(v, DeviceArray) for v in lam):
        return DeviceArray(out)
    return out.cpu().numpy()


def _local_E(systems, lam):
    """E_d of every domain of ``systems`` (recover_primal's solves), as the
    columns of E^T (r x sum n_d, domain d at column offset e_off[d])."""
    t = require_cuda()
    def x_ok(s):
        src = getattr(s, "_d3m_src", None)
        return (getattr(s, "_d3m_X", None) is not None and src is not None and src[0] is s.f
                and len(src[1]) == len(s.couplings) and all(a is c.D for a, c in zip(src[1], s.couplings))
                and src[2] == _fingerprint(s.f))

    use_x = []
    for s in systems:
        if s.factor is None:
            raise SolverStateError(f"domain {s.domain} has no cached factorization; run reduce_domain first")
        use_x.append(x_ok(s))
        if s.factor.released and not use_x[-1]:
            raise SolverStateError(f"domain {s.domain}: loads or couplings changed after reduce_domains("
                                   f"keep='solution'); reduce again")
    device_in = all(isinstance(v, DeviceArray) for v in lam)
    lam_dev = [to_device(v) for v in lam]
    r = max([int(v.shape[1]) if v.dim() == 2 else 1 for v in lam_dev] + [1])
    one_d = all(v.dim() == 1 for v in lam_dev)
    lam_dev = [v.reshape(int(v.shape[0]), r) for v in lam_dev]
    n_glob = 1 + max(int(np.max(s.dof_map)) for s in systems)
    e_off, o = [], 0
    for s in systems:
        e_off.append(o)
        o += s.n_dofs
    ET = empty((r, max(o, 1)))                    # E^T: column q of every domain contiguous

    def lam_of(s):
        parts = [lam_dev[c.interface] for c in s.couplings if np.shape(c.D)[1]]
        return t.cat(parts) if parts else t.zeros((0, r), dtype=t.complex128, device="cuda")

    # -- domains with a cached factor: batched solves per (n, m) group
    groups: dict[tuple[int, int], list[int]] = {}
    for idx, s in enumerate(systems):
        if not use_x[idx]:
            m = sum(int(np.shape(c.D)[1]) for c in s.couplings)
            groups.setdefault((s.n_dofs, m), []).append(idx)
    for (n, m), members in groups.items():
        B = len(members)
        rhs = empty((B, n, r))
        for i, idx in enumerate(members):
            rhs[i].copy_(to_device(systems[idx].f).reshape(n, r))
        F, sf = _as_batch([systems[idx].factor.packed for idx in members], (n, n))
        pv, sp = _as_batch([systems[idx].factor.perm_dev for idx in members], (n,))
        tg, st = _as_batch([systems[idx].factor.tags_dev for idx in members], (n,))
        if m:
            D, sd = _as_batch([s._d3m_D if _dev_D(s) else to_device(_coupling_matrix(s))
                               for s in (systems[idx] for idx in members)], (n, m))
            lamc = t.stack([lam_of(systems[idx]) for idx in members]).contiguous()
            tasks = np.zeros(B, dtype=_lib.GEMM_TASK)
            tasks["a_off"] = np.arange(B) * sd
            tasks["b_off"] = np.arange(B) * m * r
            tasks["c_off"] = np.arange(B) * n * r
            tasks["m"], tasks["n"], tasks["k"] = n, r, m
            tasks["lda"], tasks["ldb"], tasks["ldc"] = int(D.stride(1)), r, r
            tasks["flags"] = _lib.GEMM_SUB
            d_tasks = t.empty(64 * B, dtype=t.uint8, device="cuda")
            _lib.call("d3m_zgemm_grouped", 0, 1, _P(D), _P(lamc), _P(rhs), _lib.hptr(tasks), B, _P(d_tasks),
                      stream_ptr())
        work = empty((B, n, r))
        if n > _lib.PANEL_BK_MIN:
            d_tasks = t.empty(64 * 2 * ((n + 63) // 64) * B, dtype=t.uint8, device="cuda")
            _lib.call("d3m_ldlt_solve_blocked_batched", B, n, _P(F), sf, _P(pv), sp, _P(tg), st, _P(rhs), n * r,
                      r, r, _P(work), _P(d_tasks), stream_ptr())
        else:
            _lib.call("d3m_ldlt_solve_batched", B, n, _P(F), sf, _P(pv), sp, _P(tg), st, _P(rhs), n * r, r, r,
                      _P(work), stream_ptr())
        for i, idx in enumerate(members):
            ET[:, e_off[idx]:e_off[idx] + n].copy_(rhs[i].t())
    # -- domains reduced with keep="solution": E_d = X_F - X_D lambda_d
    sol = [idx for idx in range(len(systems)) if use_x[idx]]
    by_base: dict[int, list[int]] = {}
    for idx in sol:
        by_base.setdefault(systems[idx]._d3m_X.untyped_storage().data_ptr(), []).append(idx)
    for base, members in by_base.items():
        Xst = systems[members[0]]._d3m_X
        whole = t.empty(0, dtype=t.complex128, device="cuda").set_(
            Xst.untyped_storage(), 0, (Xst.untyped_storage().nbytes() // 16,))
        lams = [lam_of(systems[idx]) for idx in members]
        loff = np.concatenate([[0], np.cumsum([int(v.numel()) for v in lams])]).astype(np.int64)
        lamc = t.cat([v.reshape(-1) for v in lams] + [t.zeros(1, dtype=t.complex128, device="cuda")])
        goff = np.concatenate([[0], np.cumsum([systems[idx].n_dofs for idx in members])]).astype(np.int64)
        Eg = empty((int(goff[-1]), r))
        tasks = []
        for i, idx in enumerate(members):
            s = systems[idx]
            X, mp, n = s._d3m_X, s._d3m_Xm, s.n_dofs
            mr = int(lams[i].shape[0])
            Eg[int(goff[i]):int(goff[i + 1])].copy_(X[:, mp:mp + r])
            if mr:
                tk = np.zeros(1, dtype=_lib.GEMM_TASK)
                tk["a_off"] = (X.data_ptr() - base) // 16
                tk["b_off"] = loff[i]
                tk["c_off"] = goff[i] * r
                tk["m"], tk["n"], tk["k"] = n, r, mr
                tk["lda"], tk["ldb"], tk["ldc"] = int(X.stride(0)), r, r
                tk["flags"] = _lib.GEMM_SUB
                tasks.append(tk)
        if tasks:
            tk = np.concatenate(tasks)
            d_tasks = t.empty(64 * len(tk), dtype=t.uint8, device="cuda")
            _lib.call("d3m_zgemm_grouped", 0, 1, _P(whole), _P(lamc), _P(Eg), _lib.hptr(tk), len(tk),
                      _P(d_tasks), stream_ptr())
        for i, idx in enumerate(members):
            n = systems[idx].n_dofs
            ET[:, e_off[idx]:e_off[idx] + n].copy_(Eg[int(goff[i]):int(goff[i + 1])].t())
    return ET, e_off, r, one_d


def _ordered_average(systems, ET, e_off, r, n_glob=None):
    """Average of the domains' E_d over duplicated global dofs, accumulated
    per dof in ascending domain order (subdomain.py:229-237) -> r x n_glob."""
    if n_glob is None:
        n_glob = 1 + max(int(np.max(s.dof_map)) for s in systems)
    gl, src = [], []
    for idx in range(len(systems)):          # acc[dof_map] += E in list order
        dm = np.asarray(systems[idx].dof_map, dtype=np.int64)
        gl.append(dm)
        src.append(e_off[idx] + np.arange(dm.size, dtype=np.int64))
    gl = np.concatenate(gl)
    src = np.concatenate(src)
    order_ = np.argsort(gl, kind="stable")
    counts = np.bincount(gl, minlength=n_glob)
    ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    outT = empty((r, n_glob))
    d_ptr, d_src = upload_i64(ptr), upload_i64(src[order_])   # both alive across the launches
    for q in range(r):
        _lib.call("d3m_ordered_average", _P(ET[q]), _P(d_ptr), _P(d_src), _P(outT[q]), n_glob, stream_ptr())
    return outT

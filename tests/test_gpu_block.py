"""GPU parity: block LDL^T (restricted BK, DMMA trailing updates) and block
substitution vs the oracle, the reference goldens and dense solves."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, rand_complex_symmetric, split_blocks

pytestmark = pytest.mark.gpu


def _plan(K, order=None):
    import paper_2002_05018_b200 as d
    g = d.clique_graph(K)
    if order is None:
        order = d.reorder(g, K.sizes)
    return d.symbolic_factor(g, order, K.sizes)


@pytest.fixture(params=[3, 4], ids=["3m", "4m"])
def gemm_form(request, cuda):
    """Run a test under each complex product form of the grouped GEMM."""
    from paper_2002_05018_b200 import _lib
    prev = _lib.gemm_form(request.param)
    yield request.param
    _lib.gemm_form(prev)


def test_gemm_vs_numpy(cuda, gemm_form):
    """Grouped DMMA GEMM, all four operand layouts and three modes, both
    complex product forms (3M default, 4M)."""
    from paper_2002_05018_b200 import _lib
    from paper_2002_05018_b200.device import stream_ptr, to_device
    rng = np.random.default_rng(3)
    for (M, N, K) in [(64, 64, 64), (1, 1, 1), (70, 33, 130), (256, 256, 256), (129, 65, 7), (200, 190, 40), (64, 64, 32)]:
        for ta in (0, 1):
            for tb in (0, 1):
                for mode in (_lib.GEMM_SUB, _lib.GEMM_STORE, _lib.GEMM_ADD):
                    A = rng.standard_normal((M, K)) + 1j * rng.standard_normal((M, K))
                    B = rng.standard_normal((N, K)) + 1j * rng.standard_normal((N, K))
                    C = rng.standard_normal((M, N)) + 1j * rng.standard_normal((M, N))
                    As = A.T.copy() if ta else A
                    Bs = B.T.copy() if tb else B
                    dA, dB, dC = to_device(As), to_device(Bs), to_device(C)
                    task = np.zeros(1, dtype=_lib.GEMM_TASK)
                    task["m"], task["n"], task["k"] = M, N, K
                    task["lda"] = M if ta else K
                    task["ldb"] = N if tb else K
                    task["ldc"] = N
                    task["flags"] = mode
                    dt = cuda.empty(64, dtype=cuda.uint8, device="cuda")
                    _lib.call("d3m_zgemm_grouped", ta, tb, _lib.ptr(dA), _lib.ptr(dB), _lib.ptr(dC),
                              _lib.hptr(task), 1, _lib.ptr(dt), stream_ptr())
                    P = A @ B.T
                    ref = {0: C - P, 1: P, 2: C + P}[mode]
                    got = dC.cpu().numpy()
                    assert np.abs(got - ref).max() <= 1e-13 * max(1.0, np.abs(ref).max()) * K, (M, N, K, ta, tb, mode)


def test_gemm_symmetric_target(cuda, gemm_form):
    from paper_2002_05018_b200 import _lib
    from paper_2002_05018_b200.device import stream_ptr, to_device
    rng = np.random.default_rng(4)
    n, K = 150, 40
    X = rng.standard_normal((n, K)) + 1j * rng.standard_normal((n, K))
    L = rng.standard_normal((n, K)) + 1j * rng.standard_normal((n, K))
    W = rand_complex_symmetric(n, 5)
    dX, dL, dW = to_device(X), to_device(L), to_device(W)
    task = np.zeros(1, dtype=_lib.GEMM_TASK)
    task["m"] = task["n"] = n
    task["k"] = K
    task["lda"] = task["ldb"] = K
    task["ldc"] = n
    task["flags"] = _lib.GEMM_SUB | _lib.GEMM_SYM
    dt = cuda.empty(64, dtype=cuda.uint8, device="cuda")
    _lib.call("d3m_zgemm_grouped", 0, 0, _lib.ptr(dX), _lib.ptr(dL), _lib.ptr(dW), _lib.hptr(task), 1,
              _lib.ptr(dt), stream_ptr())
    upd = X @ L.T
    upd = np.tril(upd) + np.tril(upd, -1).T               # factor.py:217-220
    got = dW.cpu().numpy()
    assert np.array_equal(got, got.T)
    assert np.abs(got - (W - upd)).max() <= 1e-12 * np.abs(upd).max()


def test_gemm_3m_error_is_rounding_level(cuda):
    """Integer-valued operands keep every product and partial sum exact in
    fp64, so both product forms must reproduce A B^T exactly (this catches
    any mis-assembled 3M term, which a rounding tolerance could hide)."""
    from paper_2002_05018_b200 import _lib
    from paper_2002_05018_b200.device import stream_ptr, to_device
    rng = np.random.default_rng(9)
    M, N, K = 130, 70, 256
    A = rng.integers(-64, 64, (M, K)) + 1j * rng.integers(-64, 64, (M, K))
    B = rng.integers(-64, 64, (N, K)) + 1j * rng.integers(-64, 64, (N, K))
    exact = A @ B.T                                       # |sums| < 2^53: exact in complex128
    for form in (3, 4):
        prev = _lib.gemm_form(form)
        dA, dB, dC = to_device(A), to_device(B), to_device(np.zeros((M, N), complex))
        task = np.zeros(1, dtype=_lib.GEMM_TASK)
        task["m"], task["n"], task["k"], task["lda"], task["ldb"], task["ldc"] = M, N, K, K, K, N
        task["flags"] = _lib.GEMM_STORE
        dt = cuda.empty(64, dtype=cuda.uint8, device="cuda")
        _lib.call("d3m_zgemm_grouped", 0, 0, _lib.ptr(dA), _lib.ptr(dB), _lib.ptr(dC),
                  _lib.hptr(task), 1, _lib.ptr(dt), stream_ptr())
        _lib.gemm_form(prev)
        assert np.array_equal(dC.cpu().numpy(), exact), form


def test_block_pivots_and_solution_vs_reference_goldens(cuda):
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import workloads as wl
    g = golden("block_small.npz")
    for seed in range(30):
        K, S = wl.rand_block_system(seed, max_blocks=10, max_size=12, density=0.4)
        plan = _plan(K)
        assert np.array_equal(plan.order.perm, g[f"s{seed}_order"])
        F = d.block_ldlt(K, plan)
        assert np.array_equal(np.concatenate([f.perm for f in F.diag]), g[f"s{seed}_perm"])
        assert np.array_equal(np.concatenate([f.tags for f in F.diag]), g[f"s{seed}_tags"])
        st = g[f"s{seed}_stats"]
        assert (F.stats.factor_entries, F.stats.flops, F.stats.peak_bytes, F.stats.n_2x2_pivots) == tuple(st)
        rng = np.random.default_rng(900 + seed)
        b = rng.standard_normal((S.shape[0], 3)) + 1j * rng.standard_normal((S.shape[0], 3))
        x = np.concatenate(d.block_solve(F, split_blocks(b, K.sizes)))
        ref = g[f"s{seed}_x"]
        assert np.linalg.norm(x - ref) <= 1e-11 * np.linalg.norm(ref)
        assert np.linalg.norm(S @ x - b) <= 1e-12 * np.linalg.norm(b)


def test_block_vs_oracle_larger_blocks(cuda, oracle):
    """Pivots bit-exact vs the oracle on indefinite systems with 64-300 wide
    supernodes (tile edges, 2x2 pivots, fill)."""
    import paper_2002_05018_b200 as d
    rng = np.random.default_rng(77)
    for case in range(4):
        nb = int(rng.integers(3, 7))
        sizes = rng.integers(40, 300, size=nb)
        n = int(sizes.sum())
        off = np.concatenate([[0], np.cumsum(sizes)])
        trip = []
        for i in range(nb):
            G = rng.standard_normal((sizes[i], sizes[i])) + 1j * rng.standard_normal((sizes[i], sizes[i]))
            Dg = (np.tril(G) + np.tril(G, -1).T) / np.sqrt(2 * sizes[i])
            Dg[np.diag_indices(sizes[i])] += rng.uniform(-2, 2, sizes[i])
            trip.append((i, i, Dg))
            for j in range(i):
                if rng.random() < 0.6:
                    trip.append((i, j, (rng.standard_normal((sizes[i], sizes[j])) +
                                        1j * rng.standard_normal((sizes[i], sizes[j]))) / np.sqrt(2 * 256)))
        K = d.from_blocks(sizes, trip)
        plan = _plan(K)
        F = d.block_ldlt(K, plan)
        adj = oracle.clique_adjacency(nb, K.blocks.keys())
        op = oracle.symbolic_factor(adj, plan.order.perm, sizes)
        Fo = oracle.block_ldlt({k: np.asarray(v) for k, v in K.blocks.items()}, op)
        for j in range(nb):
            assert np.array_equal(F.diag[j].perm, Fo.diag[j].perm), (case, j)
            assert np.array_equal(F.diag[j].tags, Fo.diag[j].tags), (case, j)
        for key, Lo in Fo.offdiag.items():
            assert np.abs(F.offdiag[key] - Lo).max() <= 1e-9 * max(1.0, np.abs(Lo).max())
        B = rng.standard_normal((n, 4)) + 1j * rng.standard_normal((n, 4))
        x = np.concatenate(d.block_solve(F, split_blocks(B, sizes)))
        xo = np.concatenate(oracle.block_solve(Fo, split_blocks(B, sizes)))
        assert np.linalg.norm(x - xo) <= 1e-9 * np.linalg.norm(xo)
        S = K.scatter()
        assert np.linalg.norm(S @ x - B) <= 1e-10 * np.linalg.norm(B) * np.linalg.norm(S) * np.linalg.norm(x) / np.linalg.norm(B)


def test_reference_kats(cuda):
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import workloads as wl
    M = rand_complex_symmetric(9, 0)                        # test_block_factor.py:24-32
    K = d.from_blocks([9], [(0, 0, M)])
    F = d.block_ldlt(K, _plan(K))
    ref = d.dense_ldlt_bk(M)
    assert np.array_equal(F.diag[0].L, ref.L) and np.array_equal(F.diag[0].d, ref.d)
    assert np.array_equal(F.diag[0].perm, ref.perm) and F.offdiag == {}
    rng = np.random.default_rng(6)                          # :54-72 four-cycle fill
    sizes = [2, 3, 2, 4]

    def sym(n):
        G = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        return (G + G.T) / 2 + 3 * n * np.eye(n)
    tri = [(i, i, sym(sizes[i])) for i in range(4)]
    for (i, j) in [(1, 0), (2, 1), (3, 2), (3, 0)]:
        tri.append((i, j, rng.standard_normal((sizes[i], sizes[j])) + 0j))
    K = d.from_blocks(sizes, tri)
    plan = _plan(K, d.identity_ordering(4))
    assert d.fill_blocks(plan, d.clique_graph(K)) == [(3, 1)]
    F = d.block_ldlt(K, plan)
    assert set(F.offdiag) - {(i, j) for (i, j) in K.blocks if i != j} == {(3, 1)}
    sizes = [3, 2]                                          # :75-83 identity blocks
    K = d.from_blocks(sizes, [(0, 0, np.eye(3, dtype=complex)), (1, 1, np.eye(2, dtype=complex))])
    F = d.block_ldlt(K, _plan(K))
    gv = [np.arange(3) + 0j, np.array([5.0, 6.0]) + 1j]
    x = d.block_solve(F, gv)
    assert np.array_equal(x[0], gv[0]) and np.array_equal(x[1], gv[1])
    K = d.BlockSparseSym([])                                # :159-164 empty
    F = d.block_ldlt(K, _plan(K, d.identity_ordering(0)))
    assert d.block_solve(F, []) == [] and F.stats.factor_entries == 0
    K, _ = wl.rand_block_system(61)                         # :167-171
    F = d.block_ldlt(K, _plan(K))
    with pytest.raises(ValueError):
        d.block_solve(F, [np.ones(2, dtype=complex)] * (K.nblocks + 1))
    sizes = [2, 2]                                          # :144-149
    K = d.from_blocks(sizes, [(0, 0, np.zeros((2, 2), dtype=complex)), (1, 1, np.eye(2, dtype=complex))])
    with pytest.raises(d.SingularBlockError, match="block column 0"):
        d.block_ldlt(K, _plan(K, d.identity_ordering(2)))


@pytest.mark.parametrize("n,sym_exact", [(200, True), (256, True), (257, False), (360, True), (384, True),
                                         (447, True), (456, False), (512, True), (600, True)])
def test_cluster_diag_bk_is_bit_exact(cuda, oracle, monkeypatch, n, sym_exact):
    """Supernodes wider than 128 take the cluster-resident exact BK
    (bk_cluster.cu; 8-CTA clusters up to n = 400, 16-CTA clusters up to 526,
    the config-5 supernodes are 447-456 wide): a one-block K factors bit for
    bit like the CPU oracle (the restatement of kernels.py:36-146) and like
    dense_ldlt_bk (the single-CTA exact kernel) -- L, d, e, perm, tags,
    growth -- for the known-symmetric prologue and the full symmetry check
    alike, and for every cluster size (a size that does not fit moves to a
    larger cluster; n = 600 fits none and takes the exact kernel)."""
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import _lib
    M = rand_complex_symmetric(n, n)
    M[np.diag_indices(n)] += np.random.default_rng(n).uniform(-1, 1, n)
    if not sym_exact:       # not exactly symmetric (within 1e-12): full check path
        M[5, 3] += 1e-15 * abs(M[5, 3])
    ref = d.dense_ldlt_bk(M)
    assert ref.n_2x2 > 0
    if n >= 384:
        fo = oracle.dense_ldlt_bk(M)
        assert np.array_equal(ref.perm, fo.perm) and np.array_equal(ref.tags, fo.tags)
        assert np.array_equal(np.tril(ref.packed.cpu().numpy()), np.tril(fo.packed))
        assert ref.growth == fo.growth
    lib = _lib.load()
    assert lib.d3m_bk_cluster_max_n(16) >= 512 and lib.d3m_bk_cluster_max_n(8) >= 384
    for cs in ("16", "8", "4", "2"):
        monkeypatch.setenv("D3M_BKC_CS", cs)
        K = d.from_blocks([n], [(0, 0, M)])
        F = d.block_ldlt(K, _plan(K))
        f = F.diag[0]
        assert np.array_equal(f.perm, ref.perm) and np.array_equal(f.tags, ref.tags)
        assert np.array_equal(f.L, ref.L) and np.array_equal(f.d, ref.d) and np.array_equal(f.e, ref.e)
        assert F.stats.growth_factor == ref.growth


def test_multi_rhs_equals_single_rhs_bitwise(cuda):
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import workloads as wl
    K, _ = wl.rand_block_system(77, max_blocks=5, max_size=6)   # test_block_factor.py:109-120
    F = d.block_ldlt(K, _plan(K))
    rng = np.random.default_rng(78)
    B = [rng.standard_normal((int(s), 5)) + 1j * rng.standard_normal((int(s), 5)) for s in K.sizes]
    X = d.block_solve(F, B)
    for c in range(5):
        Xc = d.block_solve(F, [b[:, c:c + 1] for b in B])
        for i in range(K.nblocks):
            assert np.array_equal(X[i][:, c:c + 1], Xc[i])


@pytest.mark.parametrize("seed,max_blocks,max_size", [(91, 7, 60), (93, 6, 300), (95, 12, 20)])
def test_solve_kernels_bitwise_equal(cuda, monkeypatch, seed, max_blocks, max_size):
    """The dataflow block solve (default), the grid-barrier persistent kernel
    (ABI v5) and the per-product launch sequence give bitwise equal
    solutions, over two passes of RHS (20 columns); columns solved alone
    equal the multi-RHS solve bitwise."""
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import factor as fac
    from paper_2002_05018_b200 import workloads as wl
    K, _ = wl.rand_block_system(seed, max_blocks=max_blocks, max_size=max_size)
    F = d.block_ldlt(K, _plan(K))
    rng = np.random.default_rng(seed + 1)
    B = [rng.standard_normal((int(s), 20)) + 1j * rng.standard_normal((int(s), 20)) for s in K.sizes]
    assert fac._SOLVE_MODE == "flow"
    X0 = d.block_solve(F, B)
    monkeypatch.setattr(fac, "_SOLVE_MODE", "barrier")
    X1 = d.block_solve(F, B)
    monkeypatch.setattr(fac, "_solve_plan", lambda sched: None)
    X2 = d.block_solve(F, B)
    for i in range(K.nblocks):
        assert np.array_equal(X0[i], X1[i])
        assert np.array_equal(X1[i], X2[i])
    monkeypatch.undo()
    for c in (0, 15, 16, 19):
        Xc = d.block_solve(F, [b[:, c:c + 1] for b in B])
        for i in range(K.nblocks):
            assert np.array_equal(X0[i][:, c:c + 1], Xc[i])


def test_determinism(cuda):
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import workloads as wl
    K, _ = wl.rand_block_system(55, max_blocks=8, max_size=70)
    plan = _plan(K)
    F1, F2 = d.block_ldlt(K, plan), d.block_ldlt(K, plan)
    assert np.array_equal(F1._pool.cpu().numpy(), F2._pool.cpu().numpy())


@pytest.mark.slow
def test_config4_full_size_vs_reference(cuda):
    """BASELINE config 4 at full size: pivot sequence of all 144 supernodes
    bit-exact vs the reference, solution within 1e-9 of the reference's,
    residual of all 16 RHS reported against the reference's own."""
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import workloads as wl
    g = golden("cfg4.npz")
    K = wl.config4_matrix()
    plan = _plan(K, d.identity_ordering(K.nblocks))
    assert plan.total_factor_entries == int(g["pattern_total"])
    F = d.block_ldlt(K, plan)
    perm = np.stack([f.perm for f in F.diag])
    tags = np.stack([f.tags for f in F.diag])
    assert np.array_equal(perm, g["perm"].astype(np.int64))
    assert np.array_equal(tags, g["tags"])
    assert np.array_equal(np.array([f.n_2x2 for f in F.diag]), g["n2x2"])
    st = g["stats"]
    assert (F.stats.factor_entries, F.stats.flops, F.stats.peak_bytes, F.stats.n_2x2_pivots) == tuple(st)
    rhs = wl.config4_rhs(K)
    x = d.block_solve(F, rhs)
    x0 = np.concatenate([xi[:, 0] for xi in x])
    ref = g["x0"]
    assert np.linalg.norm(x0 - ref) <= 1e-9 * np.linalg.norm(ref)
    # residuals against the reference's own (tools/gen_cfg4_residuals.py):
    # the reference reaches max 1.1e-10 over the 16 RHS; the unrefined GPU
    # solve stays within a small factor of it, one refinement step goes to
    # rounding level
    gr = golden("cfg4_residuals.npz")["residual"]
    res = _block_residuals(K, rhs, x)
    assert np.all(res <= 8.0 * gr), (res, gr)
    xr = d.block_solve(F, rhs, refine=1)
    res_r = _block_residuals(K, rhs, xr)
    assert np.all(res_r <= 1e-12) and np.all(res_r < gr), res_r
    xr0 = np.concatenate([xi[:, 0] for xi in xr])
    assert np.linalg.norm(xr0 - ref) <= 1e-9 * np.linalg.norm(ref)


def _block_residuals(K, rhs, x):
    """Per RHS column: ||K x - b|| / ||b|| over the stored blocks (host)."""
    Kx = [np.zeros_like(np.asarray(b).reshape(b.shape[0], -1)) for b in rhs]
    xs = [np.asarray(v).reshape(v.shape[0], -1) for v in x]
    for (i, j), blk in K.blocks.items():
        B = np.asarray(blk)
        Kx[i] += B @ xs[j]
        if i != j:
            Kx[j] += B.T @ xs[i]
    bs = [np.asarray(b).reshape(b.shape[0], -1) for b in rhs]
    num = np.sqrt(sum(np.sum(np.abs(Kx[i] - bs[i]) ** 2, axis=0) for i in range(len(bs))))
    den = np.sqrt(sum(np.sum(np.abs(bs[i]) ** 2, axis=0) for i in range(len(bs))))
    return num / den


@pytest.mark.parametrize("device_k", [False, True])
def test_refined_solve(cuda, device_k):
    """block_solve(refine=1): residual to rounding level on an ill-conditioned
    (weak-shift) system, solution closer to the dense solve than unrefined,
    k-RHS refinement bitwise equal to k single-RHS refinements, host and
    device K alike."""
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import workloads as wl
    from paper_2002_05018_b200.factor import to_device_blocks
    K, S = wl.rand_block_system(123, max_blocks=9, max_size=60, density=0.5, shift=0.5)
    plan = _plan(K)
    F = d.block_ldlt(to_device_blocks(K) if device_k else K, plan)
    rng = np.random.default_rng(5)
    rhs = [rng.standard_normal((int(n), 3)) + 1j * rng.standard_normal((int(n), 3)) for n in K.sizes]
    x0 = d.block_solve(F, rhs)
    x1 = d.block_solve(F, rhs, refine=1)
    x2 = d.block_solve(F, rhs, refine=2)
    r0, r1, r2 = (_block_residuals(K, rhs, x) for x in (x0, x1, x2))
    assert np.all(r1 <= r0) and np.all(r1 < 1e-14), (r0, r1)
    assert np.all(r2 < 1e-14)
    xd = np.linalg.solve(S, np.concatenate(rhs))
    e0 = np.linalg.norm(np.concatenate(x0) - xd) / np.linalg.norm(xd)
    e1 = np.linalg.norm(np.concatenate(x1) - xd) / np.linalg.norm(xd)
    assert e1 <= max(e0, 1e-13), (e0, e1)
    for c in range(3):
        xc = d.block_solve(F, [b[:, c:c + 1] for b in rhs], refine=1)
        for a, b_ in zip(x1, xc):
            assert np.array_equal(a[:, c], b_[:, 0])


def test_pinned_streamed_upload_and_host_tensor_solve(cuda):
    """K given as views of one pinned host allocation takes the chunked,
    first-touch streamed upload (twice: the second call reuses the cached
    chunk plan); the factor equals the one from numpy blocks bit for bit, and
    a solve with pinned host-tensor RHS returns host tensors equal to the
    numpy-RHS solve."""
    import torch
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import workloads as wl
    K, _ = wl.rand_block_system(131, max_blocks=14, max_size=40, density=0.5)
    while K.nblocks < 10:
        K, _ = wl.rand_block_system(int(K.nblocks) + 500, max_blocks=14, max_size=40, density=0.5)
    plan = _plan(K)
    F0 = d.block_ldlt(K, plan)
    tot = sum(int(np.asarray(b).size) for b in K.blocks.values())
    buf = torch.empty(tot, dtype=torch.complex128, pin_memory=True)
    Kp = d.BlockSparseSym(K.sizes)
    o = 0
    for k, b in K.blocks.items():
        b = np.ascontiguousarray(np.asarray(b, dtype=np.complex128))
        v = buf[o:o + b.size].view(b.shape)
        v.copy_(torch.from_numpy(b))
        Kp.blocks[k] = v
        o += b.size
    sched = F0._sched
    for rep in range(2):
        F = d.block_ldlt(Kp, plan)
        assert np.array_equal(F._pool.cpu().numpy(), F0._pool.cpu().numpy()), rep
    assert len(getattr(sched, "upload_cache", {})) >= 1
    rng = np.random.default_rng(7)
    rhs = [rng.standard_normal((int(n), 3)) + 1j * rng.standard_normal((int(n), 3)) for n in K.sizes]
    x0 = d.block_solve(F0, rhs)
    xp = d.block_solve(F, [torch.from_numpy(r).pin_memory() for r in rhs])
    for a, b in zip(x0, xp):
        assert isinstance(b, torch.Tensor) and not b.is_cuda
        assert np.array_equal(a, b.numpy())


def test_concurrent_block_ldlt_from_two_threads(cuda):
    """libd3m keeps its executor state per device and serialises the enqueue
    of concurrent calls (d3m_capi.cu ExecCtx): two host threads factoring and
    solving at once (ctypes releases the GIL) get the bitwise results of the
    sequential calls."""
    import threading

    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import workloads as wl
    K, _ = wl.rand_block_system(97, max_blocks=8, max_size=300)
    plan = _plan(K)
    rng = np.random.default_rng(98)
    B = [rng.standard_normal((int(s), 3)) + 1j * rng.standard_normal((int(s), 3)) for s in K.sizes]
    F0 = d.block_ldlt(K, plan)
    x0 = [np.asarray(v) for v in d.block_solve(F0, B)]
    out, errs = {}, []

    def work(tag):
        try:
            for it in range(3):
                F = d.block_ldlt(K, plan)
                out[(tag, it)] = ([f.perm for f in F.diag], [np.asarray(v) for v in d.block_solve(F, B)])
        except Exception as e:          # noqa: BLE001  (reported below)
            errs.append(e)
    th = [threading.Thread(target=work, args=(t,)) for t in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for (perms, x) in out.values():
        for p, f in zip(perms, F0.diag):
            assert np.array_equal(p, f.perm)
        for a, b in zip(x, x0):
            assert np.array_equal(a, b)


def test_real_and_single_precision_tensor_inputs_are_converted(cuda):
    """A torch RHS of another dtype (float64, complex64) is converted like
    np.asarray(b, complex128) would convert it, not reinterpreted."""
    import torch

    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import workloads as wl
    K, _ = wl.rand_block_system(55, max_blocks=5, max_size=20)
    F = d.block_ldlt(K, _plan(K))
    rng = np.random.default_rng(56)
    Br = [rng.standard_normal(int(s)) for s in K.sizes]
    want = [np.asarray(v) for v in d.block_solve(F, [b.astype(complex) for b in Br])]
    for conv in (lambda b: torch.from_numpy(b).cuda(), lambda b: torch.from_numpy(b)):
        got = [np.asarray(v) for v in d.block_solve(F, [conv(b) for b in Br])]
        for a, b in zip(got, want):
            assert np.array_equal(a, b)
    B64 = [torch.from_numpy(b.astype(np.complex64)).cuda() for b in Br]
    got = [np.asarray(v) for v in d.block_solve(F, B64)]
    for a, b in zip(got, want):
        assert np.abs(a - b).max() <= 1e-5 * max(np.abs(b).max(), 1.0)
    f = d.dense_ldlt_bk(torch.eye(4, dtype=torch.float64, device="cuda"))
    assert np.array_equal(f.d, np.ones(4, dtype=complex))


def test_host_staged_upload_matches_device_inputs(cuda):
    """numpy K blocks (the reference API's inputs) take the host-staged
    upload (a native thread fills a pinned ring chunk by chunk, the copy
    stream waits on a pinned flag per chunk): repeated factorisations, a
    real-valued and a non-contiguous block included, equal the factorisation
    of the same K from device blocks bit for bit."""
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import workloads as wl
    from paper_2002_05018_b200.factor import to_device_blocks
    K = wl.config4_matrix(seed=123, grid=(3, 3, 3), n=24)               # 54 faces: several chunks
    k0 = next(k for k in K.blocks if k[0] != k[1])
    K.blocks[k0] = np.asfortranarray(np.asarray(K.blocks[k0]).real)      # float64, F-order
    plan = _plan(K, d.identity_ordering(K.nblocks))
    assert plan.nblocks > 16                                              # several upload chunks
    Fd = d.block_ldlt(to_device_blocks(K), plan)
    rng = np.random.default_rng(124)
    B = [rng.standard_normal(int(s)) + 0j for s in K.sizes]
    xd = [np.asarray(v) for v in d.block_solve(Fd, B)]
    for _ in range(3):
        F = d.block_ldlt(K, plan)
        for f, g in zip(F.diag, Fd.diag):
            assert np.array_equal(f.perm, g.perm) and np.array_equal(f.L, g.L)
        x = [np.asarray(v) for v in d.block_solve(F, B)]
        for a, b in zip(x, xd):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("grid,n,order", [((3, 3, 3), 64, "builtin"), ((3, 3, 2), 160, "builtin"),
                                          ((3, 3, 3), 48, "natural"), ((4, 2, 2), 32, "builtin")])
def test_etree_parallel_executor_bitwise_equals_sequential(cuda, grid, n, order):
    """The etree-parallel executor (lookahead=True: critical chains of
    independent subtrees on separate streams, bulk updates in column order on
    one stream) gives the factor and solution of the in-order executor
    (lookahead=False) bit for bit, on plans whose elimination trees have many
    leaves (builtin ordering) and on a chain (natural order)."""
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import planner
    from paper_2002_05018_b200 import workloads as wl
    K = wl.config4_matrix(seed=n + len(grid), grid=grid, n=n)
    g = d.clique_graph(K)
    o = d.reorder(g, K.sizes) if order == "builtin" else d.identity_ordering(K.nblocks)
    plan = d.symbolic_factor(g, o, K.sizes)
    sched = planner.etree_schedule(plan.etree_parent, plan.pattern).reshape(-1, 3)
    if order == "builtin":
        assert len(set(sched[:, 0])) > 1               # independent subtrees spread over streams
    F0 = d.block_ldlt(K, plan, lookahead=False)
    F1 = d.block_ldlt(K, plan, lookahead=True)
    for a, b in zip(F0.diag, F1.diag):
        assert np.array_equal(a.perm, b.perm) and np.array_equal(a.L, b.L) and np.array_equal(a.d, b.d)
    for key in F0.offdiag:
        assert np.array_equal(F0.offdiag[key], F1.offdiag[key]), key
    rng = np.random.default_rng(n)
    B = [rng.standard_normal((int(s), 2)) + 1j * rng.standard_normal((int(s), 2)) for s in K.sizes]
    for a, b in zip(d.block_solve(F0, B), d.block_solve(F1, B)):
        assert np.array_equal(np.asarray(a), np.asarray(b))


def test_host_staged_upload_under_blocking_launches(cuda):
    """With CUDA_LAUNCH_BLOCKING=1 (or a profiler serialising launches) every
    launch returns only once its kernel has finished: the staging thread must
    already be running when the copy stream's flag waits are enqueued, or the
    first wait never ends.  A subprocess factors a numpy K that way."""
    import subprocess
    import sys
    from conftest import ROOT
    code = ("import sys; sys.path.insert(0, %r)\n"
            "import paper_2002_05018_b200 as d\n"
            "from paper_2002_05018_b200 import workloads as wl\n"
            "K = wl.config4_matrix(seed=5, grid=(3, 3, 2), n=16)\n"
            "plan = d.symbolic_factor(d.clique_graph(K), d.identity_ordering(K.nblocks), K.sizes)\n"
            "for _ in range(2):\n"
            "    F = d.block_ldlt(K, plan)\n"
            "print('ok', F.stats.n_2x2_pivots)\n") % ROOT
    env = dict(__import__("os").environ, CUDA_LAUNCH_BLOCKING="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stderr[-2000:]


def test_tma_and_cp_async_update_gemm_give_the_same_factor(cuda):
    """block_ldlt with the update GEMMs on the TMA-staged kernel (default) and
    on the cp.async kernel (D3M_GEMM_TMA=0, read once per process: two
    subprocesses) produces the same factor pool, pivots and solution bit for
    bit (ragged supernodes, builtin order, lookahead on)."""
    import subprocess
    import sys
    from conftest import ROOT
    code = ("import sys, hashlib; sys.path.insert(0, %r)\n"
            "import numpy as np\n"
            "import paper_2002_05018_b200 as d\n"
            "from paper_2002_05018_b200 import workloads as wl\n"
            "K = wl.config4_matrix(seed=7, grid=(3, 3, 2), n=150)\n"
            "plan = d.symbolic_factor(d.clique_graph(K), d.reorder(d.clique_graph(K), K.sizes), K.sizes)\n"
            "F = d.block_ldlt(K, plan)\n"
            "rhs = wl.config4_rhs(K, nrhs=3)\n"
            "x = d.block_solve(F, rhs)\n"
            "h = hashlib.sha256()\n"
            "h.update(F._pool.cpu().numpy().tobytes())\n"
            "for b in x: h.update(np.ascontiguousarray(np.asarray(b)).tobytes())\n"
            "print('sha', h.hexdigest(), F.stats.n_2x2_pivots)\n") % ROOT
    out = []
    for tma in ("1", "0"):
        env = dict(__import__("os").environ, D3M_GEMM_TMA=tma)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0 and r.stdout.startswith("sha"), r.stderr[-2000:]
        out.append(r.stdout.strip())
    assert out[0] == out[1]

"""The CPU oracle (oracle/) pinned against golden vectors produced by running
the reference itself (tools/gen_golden.py) and against the reference's own
known-answer tests.  CPU only."""

from __future__ import annotations

import hashlib
import math

import numpy as np
import pytest

from conftest import golden, rand_complex_symmetric

import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))


def _dense_cases():
    from gen_golden_inputs import dense_suite
    return dense_suite()


def test_bk_alpha_constant(oracle):
    # pkg/tests/test_dense_factor.py:12-13
    assert oracle.lib().d3m_oracle_bk_alpha() == (1.0 + math.sqrt(17.0)) / 8.0


def test_identity_and_swap_kats(oracle):
    # pkg/tests/test_dense_factor.py:16-31
    f = oracle.dense_ldlt_bk(np.eye(4, dtype=complex))
    assert np.array_equal(f.L, np.eye(4)) and np.array_equal(f.d, np.ones(4))
    assert np.array_equal(f.perm, np.arange(4)) and f.n_2x2 == 0
    M = np.array([[0.0, 1.0], [1.0, 0.0]], dtype=complex)
    f = oracle.dense_ldlt_bk(M)
    assert f.n_2x2 == 1 and list(f.tags) == [2, 0]
    assert np.array_equal(f.L, np.eye(2)) and np.array_equal(f.dense_d(), M)


def test_oracle_bk_bit_exact_vs_reference_goldens(oracle):
    g = golden("dense_bk.npz")
    cases = _dense_cases()
    offs = np.concatenate([[0], np.cumsum(g["sizes"])])
    for k, (name, M) in enumerate(cases):
        assert g["names"][k] == name
        W = np.array(M, dtype=np.complex128, order="C")
        sc = np.abs(W).max()
        assert sc == g["scale"][k]
        perm, tags, n2, gr, info = oracle.bk_factor(W, 1e-12 * sc)
        assert np.array_equal(perm, g["perm"][offs[k]:offs[k + 1]]), name
        assert np.array_equal(tags, g["tags"][offs[k]:offs[k + 1]]), name
        assert n2 == g["n2x2"][k] and info == g["info"][k] and gr == g["growth"][k], name
        assert hashlib.sha256(np.tril(W).tobytes()).hexdigest() == g["digest"][k], name


def test_oracle_block_ldlt_vs_reference_goldens(oracle):
    from paper_2002_05018_b200 import workloads as wl
    g = golden("block_small.npz")
    for seed in range(30):
        K, S = wl.rand_block_system(seed, max_blocks=10, max_size=12, density=0.4)
        adj = oracle.clique_adjacency(K.nblocks, K.blocks.keys())
        perm = oracle.reorder(adj, K.sizes)
        assert np.array_equal(perm, g[f"s{seed}_order"])
        plan = oracle.symbolic_factor(adj, perm, K.sizes)
        F = oracle.block_ldlt({k: np.asarray(v) for k, v in K.blocks.items()}, plan)
        assert np.array_equal(np.concatenate([f.perm for f in F.diag]), g[f"s{seed}_perm"])
        assert np.array_equal(np.concatenate([f.tags for f in F.diag]), g[f"s{seed}_tags"])
        st = g[f"s{seed}_stats"]
        assert F.stats["factor_entries"] == st[0] and F.stats["flops"] == st[1]
        assert F.stats["n_2x2_pivots"] == st[3]
        rng = np.random.default_rng(900 + seed)
        b = rng.standard_normal((S.shape[0], 3)) + 1j * rng.standard_normal((S.shape[0], 3))
        off = np.concatenate([[0], np.cumsum(K.sizes)])
        x = np.concatenate(oracle.block_solve(F, [b[off[i]:off[i + 1]] for i in range(K.nblocks)]))
        ref = g[f"s{seed}_x"]
        assert np.linalg.norm(x - ref) <= 1e-13 * np.linalg.norm(ref)


def test_oracle_planning_vs_reference_goldens(oracle):
    g = golden("planning.npz")
    for c in range(int(g["count"])):
        n = int(g[f"g{c}_n"])
        adj = [set() for _ in range(n)]
        for a, b in g[f"g{c}_edges"]:
            adj[a].add(b)
            adj[b].add(a)
        w = g[f"g{c}_w"]
        perm = oracle.reorder(adj, w)
        assert np.array_equal(perm, g[f"g{c}_perm"])
        plan = oracle.symbolic_factor(adj, perm, w)
        assert np.array_equal(plan["parent"], g[f"g{c}_parent"])
        flat = np.concatenate([[len(p)] + list(p) for p in plan["pattern"]]).astype(np.int64)
        assert np.array_equal(flat, g[f"g{c}_pattern"])
        assert plan["total"] == int(g[f"g{c}_total"])


def test_oracle_ddm_vs_reference_goldens(oracle):
    from paper_2002_05018_b200 import workloads as wl
    g = golden("ddm_small.npz")
    for case, (grid, interior, fd, seed) in enumerate([((2, 2, 1), 12, 5, 0), ((3, 2, 2), 10, 4, 1)]):
        systems, part, n_glob = wl.synthetic_d3m(grid, interior, fd, seed)
        red, facs = [], []
        for d, s in enumerate(systems):
            D_all = np.concatenate([c.D for c in s.couplings], axis=1)
            K_D, g_d, fac = oracle.reduce_domain(s.A, D_all, s.f)
            assert np.array_equal(fac.perm, g[f"c{case}_fperm{d}"])
            assert np.array_equal(fac.tags, g[f"c{case}_ftags{d}"])
            ref = g[f"c{case}_KD{d}"]
            assert np.abs(K_D - ref).max() <= 1e-13 * np.abs(ref).max()
            red.append((K_D, g_d))
            facs.append(fac)
        sizes = [it.nodes.size for it in part.interfaces]
        incident = [part.incident_interfaces(d) for d in range(part.n_domains)]
        blocks, gvec = oracle.assemble_reduced(red, incident, sizes)
        adj = oracle.clique_adjacency(len(sizes), blocks.keys())
        perm = oracle.reorder(adj, sizes)
        assert np.array_equal(perm, g[f"c{case}_order"])
        plan = oracle.symbolic_factor(adj, perm, sizes)
        F = oracle.block_ldlt(blocks, plan)
        lam = oracle.block_solve(F, gvec)
        ref = g[f"c{case}_lam"]
        assert np.linalg.norm(np.concatenate(lam) - ref) <= 1e-12 * np.linalg.norm(ref)
        sol = oracle.recover_primal(facs, [s.f for s in systems],
                                    [[(c.interface, c.D) for c in s.couplings] for s in systems],
                                    [s.dof_map for s in systems], lam)
        ref = g[f"c{case}_sol"]
        assert np.linalg.norm(sol - ref) <= 1e-12 * np.linalg.norm(ref)


def test_oracle_modulus_is_glibc_hypot(oracle):
    import ctypes
    libm = ctypes.CDLL("libm.so.6")
    libm.hypot.restype = ctypes.c_double
    libm.hypot.argtypes = [ctypes.c_double, ctypes.c_double]
    rng = np.random.default_rng(5)
    x = rng.standard_normal(20000) * np.exp(rng.uniform(-700, 700, 20000))
    y = rng.standard_normal(20000) * np.exp(rng.uniform(-700, 700, 20000))
    h = oracle.hypot_array(x, y)
    for k in range(0, 20000, 7):
        assert h[k] == libm.hypot(x[k], y[k])


def test_oracle_vs_live_reference_if_present(oracle):
    """When the reference tree is mounted (build container), cross-check the
    oracle kernels against the live numba kernels on fresh random inputs."""
    from conftest import reference_available
    if not reference_available():
        pytest.skip("reference not mounted (GPU box); goldens cover this")
    import os
    import sys
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, "/root/reference/pkg/src")
    from ddsolve import kernels
    rng = np.random.default_rng(123)
    for t in range(40):
        n = int(rng.integers(1, 50))
        M = rand_complex_symmetric(n, int(rng.integers(1 << 30)))
        if t % 3 == 0:
            M[np.diag_indices(n)] = 0
        tol = 1e-12 * np.abs(M).max()
        W1, W2 = M.copy(), M.copy()
        r1, r2 = kernels.bk_factor(W1, tol), oracle.bk_factor(W2, tol)
        assert all(np.array_equal(a, b) for a, b in zip(r1[:2], r2[:2])) and r1[2:] == tuple(r2[2:])
        assert np.array_equal(np.tril(W1).view(np.int64), np.tril(W2).view(np.int64))

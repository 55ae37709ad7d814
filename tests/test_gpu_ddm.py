"""GPU parity of the DDM layer: batched Schur reduction, device assembly,
end-to-end D3M solve and recovery vs the reference goldens and dense
oracles (pkg/tests/test_subdomain.py recipes)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def _pipeline(systems, part):
    import paper_2002_05018_b200 as d
    red = d.reduce_domains(systems)
    R = d.assemble_reduced(red, part)
    g = d.clique_graph(R.K)
    order = d.reorder(g, R.K.sizes)
    plan = d.symbolic_factor(g, order, R.K.sizes)
    F = d.block_ldlt(R.K, plan)
    lam = d.block_solve(F, R.g)
    sol = d.recover_primal(systems, lam)
    return red, R, plan, F, lam, sol


def test_diagonal_example(cuda):
    import paper_2002_05018_b200 as d
    s = d.SubdomainSystem(0, np.diag([2.0, 2.0]).astype(complex), np.zeros(2, dtype=complex),
                          np.array([0, 1]), [d.Coupling(0, np.array([[1.0], [1.0]], dtype=complex), 1)])
    K_D, g_d = d.reduce_domain(s)                            # test_subdomain.py:133-143
    assert K_D.shape == (1, 1) and abs(K_D[0, 0] - 1.0) < 1e-15 and g_d[0] == 0.0
    assert isinstance(s.factor, d.DenseFactor)


def test_random_domain_vs_explicit_inverse(cuda):
    import paper_2002_05018_b200 as d
    rng = np.random.default_rng(8)                           # :154-169
    n, nl = 20, 5
    G = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    A = (G + G.T) / 2 + (2 * n) * np.eye(n)
    D = rng.standard_normal((n, nl)) + 1j * rng.standard_normal((n, nl))
    f = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    K_D, g_d = d.reduce_domain(d.SubdomainSystem(0, A, f, np.arange(n), [d.Coupling(0, D, 1)]))
    K_D, g_d = np.asarray(K_D), np.asarray(g_d)
    Ainv = np.linalg.inv(A)
    K_ref = D.T @ Ainv @ D
    assert np.abs(K_D - K_D.T).max() == 0.0
    assert np.abs(K_D - K_ref).max() <= 1e-12 * np.abs(K_ref).max()
    assert np.abs(g_d - D.T @ (Ainv @ f)).max() <= 1e-12 * np.abs(g_d).max()


def test_singular_domain_names_domain(cuda):
    import paper_2002_05018_b200 as d
    s = d.SubdomainSystem(3, np.zeros((2, 2), dtype=complex), np.zeros(2, dtype=complex), np.arange(2), [])
    with pytest.raises(d.SingularDomainError, match="domain 3"):
        d.reduce_domain(s)
    with pytest.raises(d.SolverStateError):
        d.recover_primal([d.SubdomainSystem(0, np.eye(2, dtype=complex), np.zeros(2, dtype=complex),
                                            np.arange(2), [])], [])


@pytest.mark.parametrize("case", [0, 1])
def test_pipeline_vs_reference_goldens(cuda, case):
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import workloads as wl
    g = golden("ddm_small.npz")
    grid, interior, fd, seed = [((2, 2, 1), 12, 5, 0), ((3, 2, 2), 10, 4, 1)][case]
    systems, part, n_glob = wl.synthetic_d3m(grid, interior, fd, seed)
    assert np.array_equal(np.concatenate(d.interface_lambda_nodes(part)), g[f"c{case}_kept"])
    red, R, plan, F, lam, sol = _pipeline(systems, part)
    for k, (KD, gd) in enumerate(red):
        ref = g[f"c{case}_KD{k}"]
        assert np.array_equal(systems[k].factor.perm, g[f"c{case}_fperm{k}"])
        assert np.array_equal(systems[k].factor.tags, g[f"c{case}_ftags{k}"])
        assert np.abs(np.asarray(KD) - ref).max() <= 1e-12 * np.abs(ref).max()
        assert np.abs(np.asarray(gd) - g[f"c{case}_gd{k}"]).max() <= 1e-12 * np.abs(ref).max()
    assert np.array_equal(plan.order.perm, g[f"c{case}_order"])
    lam_c = np.concatenate([np.asarray(v) for v in lam])
    ref = g[f"c{case}_lam"]
    assert np.linalg.norm(lam_c - ref) <= 1e-9 * np.linalg.norm(ref)
    ref = g[f"c{case}_sol"]
    assert np.linalg.norm(np.asarray(sol) - ref) <= 1e-9 * np.linalg.norm(ref)


def test_lambda_vs_dense_saddle_solve(cuda):
    """Oracle of test_subdomain.py:345-372: solve [[A, D], [D^T, 0]] densely."""
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import workloads as wl
    systems, part, n_glob = wl.synthetic_d3m((2, 2, 2), 9, 4, 7)
    red, R, plan, F, lam, sol = _pipeline(systems, part)
    sizes = R.interface_sizes
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(int)
    nl = int(off[-1])
    doff = np.concatenate([[0], np.cumsum([s.n_dofs for s in systems])]).astype(int)
    npr = int(doff[-1])
    S = np.zeros((npr + nl, npr + nl), dtype=complex)
    rhs = np.zeros(npr + nl, dtype=complex)
    for k, s in enumerate(systems):
        sl = slice(doff[k], doff[k + 1])
        S[sl, sl] = np.asarray(s.A)
        rhs[sl] = s.f
        for c in s.couplings:
            cl = slice(npr + off[c.interface], npr + off[c.interface + 1])
            S[sl, cl] = np.asarray(c.D)
            S[cl, sl] = c.D.T
    x = np.linalg.solve(S, rhs)
    lam_c = np.concatenate([np.asarray(v) for v in lam])
    assert np.linalg.norm(lam_c - x[npr:]) <= 1e-9 * np.linalg.norm(x[npr:])


def test_assemble_size_mismatch(cuda):
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import workloads as wl
    systems, part, _ = wl.synthetic_d3m((2, 1, 1), 6, 3, 2)
    red = d.reduce_domains(systems)
    bad = (np.asarray(red[0][0])[:-1, :-1], np.asarray(red[0][1])[:-1])
    with pytest.raises(ValueError, match="domain 0"):
        d.assemble_reduced([bad, red[1]], part)


@pytest.mark.slow
@pytest.mark.parametrize("keep", ["factor", "schur"])
def test_config3_pivots_and_schur_vs_reference(cuda, keep):
    """BASELINE config 3 subdomains (n=2048, m=384): the GPU pivot sequence is
    bit-exact with the reference's and K_D matches to 1e-9 relative -- with
    the X-based reduction and the forward-only Schur form alike."""
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import workloads as wl
    g = golden("cfg3.npz")
    doms = [int(i) for i in g["domains"]]
    systems = [d.SubdomainSystem(i, *[wl.config3_domain(i)[k] for k in (0, 2)], np.arange(2048),
                                 [d.Coupling(0, wl.config3_domain(i)[1], 1)]) for i in doms]
    red = d.reduce_domains(systems, keep=keep)
    for s, (KD, gd) in zip(systems, red):
        i = s.domain
        assert np.array_equal(s.factor.perm, g[f"perm{i}"].astype(np.int64))
        assert np.array_equal(s.factor.tags, g[f"tags{i}"])
        assert s.factor.n_2x2 == int(g[f"n2x2_{i}"])
        KDh = np.asarray(KD)
        assert abs(np.linalg.norm(KDh) - float(g[f"KDnorm{i}"])) <= 1e-9 * float(g[f"KDnorm{i}"])
        if f"KD{i}" in g.files:
            ref = g[f"KD{i}"]
            assert np.linalg.norm(KDh - ref) <= 1e-9 * np.linalg.norm(ref)


@pytest.mark.parametrize("n,m,batch,cs,nb", [(600, 40, 3, None, None), (1030, 17, 2, None, None),
                                             (600, 40, 3, "1", None), (777, 9, 2, "2", None),
                                             (777, 9, 2, "4", None), (1030, 17, 2, "8", None),
                                             (1030, 17, 2, None, "128"), (777, 9, 2, "4", "128")])
def test_large_subdomain_panel_bk_vs_oracle(cuda, oracle, monkeypatch, n, m, batch, cs, nb):
    """n > 512 takes the batched panel BK (grouped DMMA trailing updates) and
    the blocked solves: pivots bit-exact vs the oracle, K_D / g_d to 1e-10,
    for every cluster size of the panel kernel (D3M_PANEL_CS) and the 64- and
    128-column panels (D3M_PANEL_NB; 128 is the default from n = 8192)."""
    import paper_2002_05018_b200 as d
    if cs is not None:
        monkeypatch.setenv("D3M_PANEL_CS", cs)
    if nb is not None:
        monkeypatch.setenv("D3M_PANEL_NB", nb)
    rng = np.random.default_rng(n + m)
    systems, ref = [], []
    for b in range(batch):
        G = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(2 * n)
        A = (G + G.T) / 2
        A[np.diag_indices(n)] += rng.uniform(-1, 1, n) + 1j * rng.uniform(-0.1, 0.1, n)
        D = np.zeros((n, m), dtype=complex)
        D[rng.choice(n, m, replace=False), np.arange(m)] = rng.choice([-1.0, 1.0], m)
        D[:, :3] += rng.standard_normal((n, 3)) * 0.1          # some dense columns too
        f = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        systems.append(d.SubdomainSystem(b, A, f, np.arange(n), [d.Coupling(0, D, 1)]))
        ref.append(oracle.reduce_domain(A, D, f))
    red = d.reduce_domains(systems)
    for s, (KD, gd), (Ko, go, fo) in zip(systems, red, ref):
        assert np.array_equal(s.factor.perm, fo.perm)
        assert np.array_equal(s.factor.tags, fo.tags)
        assert s.factor.n_2x2 == fo.n_2x2 and fo.n_2x2 > 0
        assert 1.0 <= s.factor.growth <= 2.57
        assert np.linalg.norm(np.asarray(KD) - Ko) <= 1e-10 * np.linalg.norm(Ko)
        assert np.linalg.norm(np.asarray(gd) - go) <= 1e-10 * np.linalg.norm(go)
        # DenseFactor.solve on the large factor (blocked path)
        B = rng.standard_normal((n, 3)) + 1j * rng.standard_normal((n, 3))
        X = s.factor.solve(B)
        Xo = fo.solve(B)
        assert np.linalg.norm(X - Xo) <= 1e-10 * np.linalg.norm(Xo)


@pytest.mark.parametrize("n,batch,cs,nb", [(600, 3, None, "64"), (1030, 2, "8", "64"), (777, 2, "4", "128"),
                                           (1100, 2, None, "128")])
def test_panel_bk_tma_updates_are_bitwise_the_grouped_kernel(cuda, monkeypatch, n, batch, cs, nb):
    """The panel BK's trailing updates through the TMA-staged kernel
    (D3M_PANEL_TMA=1: per-matrix tensor maps over W and the X workspace, zeroed
    slice tail after an (NB-1)-column panel, running maximum) give the packed
    factor, pivots and growth of the cp.async grouped kernel bit for bit."""
    import paper_2002_05018_b200 as d
    if cs is not None:
        monkeypatch.setenv("D3M_PANEL_CS", cs)
    monkeypatch.setenv("D3M_PANEL_NB", nb)
    rng = np.random.default_rng(7 * n)
    mats = []
    for b in range(batch):
        G = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(2 * n)
        A = (G + G.T) / 2
        A[np.diag_indices(n)] += rng.uniform(-1, 1, n) + 1j * rng.uniform(-0.1, 0.1, n)
        mats.append(A)
    D = np.zeros((n, 2), dtype=complex)
    D[[1, n - 2], [0, 1]] = 1.0
    out = {}
    for tma in ("0", "1"):
        monkeypatch.setenv("D3M_PANEL_TMA", tma)
        systems = [d.SubdomainSystem(b, A.copy(), np.ones(n, complex), np.arange(n), [d.Coupling(0, D, 1)])
                   for b, A in enumerate(mats)]
        d.reduce_domains(systems)
        out[tma] = [(s.factor.packed.cpu().numpy(), np.asarray(s.factor.perm), np.asarray(s.factor.tags),
                     s.factor.growth, s.factor.n_2x2) for s in systems]
    for (W0, p0, t0, g0, c0), (W1, p1, t1, g1, c1) in zip(out["0"], out["1"]):
        assert c0 == c1 and c0 > 0 and g0 == g1
        assert np.array_equal(p0, p1) and np.array_equal(t0, t1)
        assert np.array_equal(np.tril(W0), np.tril(W1))


def test_padded_coupling_columns_are_skipped_exactly(cuda, oracle):
    """Domains of one batch with different coupling widths: the narrower D is
    zero-padded to the batch's m and the blocked solves skip its padded
    columns (d3m_schur_reduce_batched h_mcols, ABI v13) -- K_D, g_d and the
    recovered field match the oracle as for an unpadded domain."""
    import paper_2002_05018_b200 as d
    n = 700
    rng = np.random.default_rng(77)
    systems, ref = [], []
    for b, m in enumerate((70, 9, 33)):
        G = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(2 * n)
        A = (G + G.T) / 2
        A[np.diag_indices(n)] += rng.uniform(-1, 1, n) + 1j * rng.uniform(-0.1, 0.1, n)
        D = np.zeros((n, m), dtype=complex)
        D[rng.choice(n, m, replace=False), np.arange(m)] = rng.choice([-1.0, 1.0], m)
        f = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        systems.append(d.SubdomainSystem(b, A, f, np.arange(n), [d.Coupling(b, D, 1)]))
        ref.append(oracle.reduce_domain(A, D, f))
    red = d.reduce_domains(systems)
    for s, (KD, gd), (Ko, go, fo) in zip(systems, red, ref):
        assert np.asarray(KD).shape == Ko.shape
        assert np.array_equal(s.factor.perm, fo.perm) and np.array_equal(s.factor.tags, fo.tags)
        assert np.linalg.norm(np.asarray(KD) - Ko) <= 1e-10 * np.linalg.norm(Ko)
        assert np.linalg.norm(np.asarray(gd) - go) <= 1e-10 * np.linalg.norm(go)
        X = np.asarray(s._d3m_X.cpu().numpy() if hasattr(s._d3m_X, "cpu") else s._d3m_X)
        m = Ko.shape[0]
        assert not np.any(X[:, m:-1])                       # padded columns: exactly zero


@pytest.mark.parametrize("n,m,batch", [(600, 40, 3), (1030, 17, 2), (1296, 130, 2)])
def test_blocked_solve_tma_updates_are_bitwise_the_grouped_kernel(cuda, monkeypatch, n, m, batch):
    """The blocked subdomain solves' GEMM updates through the TMA-staged kernel
    (factor rows as row boxes, the right-hand sides and the transposed factor
    as k-major boxes; ragged last blocks stay on the cp.async kernel) give the
    Schur blocks and the kept solution of D3M_SOLVE_TMA=0 bit for bit."""
    import paper_2002_05018_b200 as d
    rng = np.random.default_rng(11 * n + m)
    mats = []
    for b in range(batch):
        G = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(2 * n)
        A = (G + G.T) / 2
        A[np.diag_indices(n)] += rng.uniform(-1, 1, n) + 1j * rng.uniform(-0.1, 0.1, n)
        D = np.zeros((n, m), dtype=complex)
        D[rng.choice(n, m, replace=False), np.arange(m)] = rng.choice([-1.0, 1.0], m)
        D[:, :2] += rng.standard_normal((n, 2)) * 0.1
        mats.append((A, D, rng.standard_normal(n) + 1j * rng.standard_normal(n)))
    out = {}
    for tma in ("0", "1"):
        monkeypatch.setenv("D3M_SOLVE_TMA", tma)
        for keep in ("factor", "schur"):
            systems = [d.SubdomainSystem(b, A.copy(), f.copy(), np.arange(n), [d.Coupling(0, D.copy(), 1)])
                       for b, (A, D, f) in enumerate(mats)]
            red = d.reduce_domains(systems, keep=keep)
            out[tma, keep] = [(np.asarray(KD), np.asarray(gd)) for KD, gd in red]
            if keep == "factor":
                B = np.arange(n * 3, dtype=float).reshape(n, 3) / n + 0.5j
                out[tma, "solve"] = [np.asarray(s.factor.solve(B)) for s in systems]
    for keep in ("factor", "schur"):
        for (K0, g0), (K1, g1) in zip(out["0", keep], out["1", keep]):
            assert np.array_equal(K0, K1) and np.array_equal(g0, g1)
    for X0, X1 in zip(out["0", "solve"], out["1", "solve"]):
        assert np.array_equal(X0, X1)


@pytest.mark.parametrize("cells,parts,radius", [(4, (2, 2, 2), 0.15), (8, (2, 1, 1), 0.0)])
def test_fem3d_pipeline_vs_monolithic(cuda, cells, parts, radius):
    """Full GPU D3M pipeline on the 3-D Nedelec problems (config 1 is the
    (8, 2x1x1) case, n = 2196 per subdomain -> panel BK path) against the
    monolithic sparse solve (test_subdomain.py:277-289 criteria)."""
    import scipy.sparse.linalg as spla
    from paper_2002_05018_b200 import fem3d
    model = fem3d.build_model(fem3d.FemProblem(cells, 0.5, parts, sphere_radius=radius))
    A, f = fem3d.assemble_global(model)
    u = spla.spsolve(A.tocsc(), f[:, 0])
    sol, systems, R, plan, F = fem3d.solve_d3m(model)
    assert np.linalg.norm(sol - u) / np.linalg.norm(u) <= 1e-8
    assert fem3d.global_residual(model, sol) <= 1e-10


@pytest.mark.slow
def test_fem3d_config2_vs_monolithic(cuda):
    """BASELINE configs[1]: 16^3 x 6 tets (31,024 edges), eps_r = 4 sphere,
    2x2x2 subdomains of 4,184 edges, lambda = 2,448."""
    import scipy.sparse.linalg as spla
    from paper_2002_05018_b200 import fem3d
    model = fem3d.build_model(fem3d.config2())
    sol, systems, R, plan, F = fem3d.solve_d3m(model)
    assert R.n_lambda == 2448
    A, f = fem3d.assemble_global(model)
    u = spla.spsolve(A.tocsc(), f[:, 0])
    assert np.linalg.norm(sol - u) / np.linalg.norm(u) <= 1e-8
    assert fem3d.global_residual(model, sol) <= 1e-10


@pytest.mark.parametrize("case", [0, 1])
def test_fem_pipeline_vs_reference_goldens(cuda, case):
    """The full GPU pipeline on 3-D Nedelec models against the REFERENCE run on
    the same systems (tools/gen_golden.py gen_fem): subdomain pivots and the
    reduced-system order / block pivots bit-exact, K_D to 1e-10, lambda and
    the recovered field to 1e-9 (case 1: n = 698 per subdomain, panel path)."""
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import fem3d
    from test_fem3d import FEM_GOLDEN_CASES
    g = golden("fem_small.npz")
    model = fem3d.build_model(fem3d.FemProblem(**FEM_GOLDEN_CASES[case]))
    systems = fem3d.subdomain_systems(model, rhs=0)
    red = d.reduce_domains(systems)
    for dd, s in enumerate(systems):
        assert np.array_equal(s.factor.perm, g[f"c{case}_fperm{dd}"])
        assert np.array_equal(s.factor.tags, g[f"c{case}_ftags{dd}"])
        KD, ref = np.asarray(red[dd][0]), g[f"c{case}_KD{dd}"]
        assert np.linalg.norm(KD - ref) <= 1e-10 * np.linalg.norm(ref)
    R = d.assemble_reduced(red, model)
    gr = d.clique_graph(R.K)
    order = d.reorder(gr, R.K.sizes)
    assert np.array_equal(order.perm, g[f"c{case}_order"])
    plan = d.symbolic_factor(gr, order, R.K.sizes)
    F = d.block_ldlt(R.K, plan)
    assert np.array_equal(np.concatenate([f.perm for f in F.diag]), g[f"c{case}_bperm"])
    lam = d.block_solve(F, R.g)
    lam_c = np.concatenate([np.asarray(v) for v in lam])
    assert np.linalg.norm(lam_c - g[f"c{case}_lam"]) <= 1e-9 * np.linalg.norm(g[f"c{case}_lam"])
    sol = np.asarray(d.recover_primal(systems, lam))
    assert np.linalg.norm(sol - g[f"c{case}_sol"]) <= 1e-9 * np.linalg.norm(g[f"c{case}_sol"])


@pytest.mark.parametrize("n,m,B", [(1, 1, 1), (37, 5, 3), (700, 45, 4), (2100, 300, 2)])
def test_nonzero_rows_vs_numpy(cuda, n, m, B):
    """d3m_nonzero_rows (the DᵀX row list): every domain's nonzero rows in
    ascending order, -1 padded to the batch maximum; an all-zero domain and
    rows whose only nonzero is the last column or has a zero real part are
    included."""
    from paper_2002_05018_b200.subdomain import _nonzero_rows
    from paper_2002_05018_b200.device import to_device
    rng = np.random.default_rng(n + m + B)
    D = np.zeros((B, n, m), dtype=np.complex128)
    for b in range(1, B):                     # domain 0 stays all-zero
        rows = rng.choice(n, size=max(1, n // 7), replace=False)
        for r in rows:
            c = int(rng.integers(0, m))
            D[b, r, c] = rng.choice([1.0, -1.0, 1j])
        D[b, rows[0], m - 1] = 1j
    idx, nrows = _nonzero_rows(to_device(D), n)
    expect = [np.flatnonzero(np.any(D[b] != 0, axis=1)) for b in range(B)]
    mx = max(len(e) for e in expect)
    if mx == 0 or mx > 0.6 * n:
        assert idx is None and nrows == 0
        return
    assert nrows == mx
    got = idx.cpu().numpy()
    for b in range(B):
        want = np.full(mx, -1, dtype=np.int64)
        want[:len(expect[b])] = expect[b]
        assert np.array_equal(got[b], want), b


def test_recover_sees_in_place_load_edits(cuda):
    """recover_primal reuses X = A^-1 [D | F] only while the loads are
    unchanged: an in-place edit of f (same object) falls back to the factor
    solve and gives the recovery of the new load."""
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import workloads as wl
    systems, part, _ = wl.synthetic_d3m((2, 2, 1), 10, 4, 3)
    red = d.reduce_domains(systems, keep="factor")
    R = d.assemble_reduced(red, part)
    gr = d.clique_graph(R.K)
    F = d.block_ldlt(R.K, d.symbolic_factor(gr, d.reorder(gr, R.K.sizes), R.K.sizes))
    lam = d.block_solve(F, R.g)
    before = np.asarray(d.recover_primal(systems, lam))
    systems[1].f[:] *= 2.0                       # in place: same object, new content
    after = np.asarray(d.recover_primal(systems, lam))
    fresh = [d.SubdomainSystem(s.domain, s.A, s.f.copy(), s.dof_map, s.couplings) for s in systems]
    d.reduce_domains(fresh, keep="factor")
    want = np.asarray(d.recover_primal(fresh, lam))
    assert not np.allclose(after, before)
    assert np.linalg.norm(after - want) <= 1e-10 * np.linalg.norm(want)


def test_config3_all_64_subdomains_vs_reference(cuda):
    """BASELINE configs[2] in full: all 64 subdomains (n = 2048, m = 384)
    reduced in one batch (panel BK, Schur-only form as the bench runs it):
    every pivot sequence (perm, tags, n2x2) equals the reference's
    (tools/gen_golden_femscale.py cfg3all, the reference's reduce_domain on
    each subdomain), K_D norms and first rows within 1e-10."""
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import workloads as wl
    g = golden("cfg3_all.npz")
    systems = wl.config3_systems(64)
    red = d.reduce_domains(systems, keep="schur", margins=True)
    for i, s in enumerate(systems):
        assert np.array_equal(s.factor.perm, g["perm"][i].astype(np.int64)), i
        assert np.array_equal(s.factor.tags, g["tags"][i]), i
        assert s.factor.n_2x2 == int(g["n2x2"][i]), i
        KD = np.asarray(red[i][0])
        assert abs(np.linalg.norm(KD) - g["KDnorm"][i]) <= 1e-10 * g["KDnorm"][i], i
        assert np.linalg.norm(KD[:8] - g["KDrows"][i]) <= 1e-10 * np.linalg.norm(g["KDrows"][i]), i
    assert min(s.factor.margin[0] for s in systems) > 1e-10

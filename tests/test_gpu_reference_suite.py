"""GPU restatement of the reference's own hot-path test suite:
block-factor residuals / reconstruction / stats (test_block_factor.py),
the acceptance criterion-4 systems (test_acceptance.py:100-119), error texts
for singular blocks and subdomains on every kernel path, 2x2 tag adjacency
(test_dense_factor.py:145-158) and the exact two-domain sum
(test_subdomain.py:188-198)."""
import numpy as np
import pytest

from conftest import rand_complex_symmetric, split_blocks

pytestmark = pytest.mark.gpu


def _plan(K, order=None):
    import paper_2002_05018_b200 as d
    g = d.clique_graph(K)
    if order is None:
        order = d.reorder(g, K.sizes)
    return d.symbolic_factor(g, order, K.sizes)


def _scalar_perm(plan):
    """Scalar permutation of the block order (plan position j holds original
    block order.perm[j])."""
    sizes = np.asarray(plan.sizes_perm)
    orig_sizes = np.zeros(plan.nblocks, dtype=np.int64)
    orig_sizes[np.asarray(plan.order.perm)] = sizes
    ooff = np.concatenate([[0], np.cumsum(orig_sizes)])
    return np.concatenate([np.arange(ooff[b], ooff[b + 1]) for b in np.asarray(plan.order.perm)]).astype(np.int64)


def test_random_block_systems_residual_reconstruction_stats(cuda):
    """test_block_factor.py:86-129: residual <= 1e-12 on 10 random systems,
    reconstruction <= 1e-11, factor_entries == the plan's prediction."""
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import workloads as wl
    for seed in range(10):
        K, S = wl.rand_block_system(seed)
        plan = _plan(K)
        F = d.block_ldlt(K, plan)
        assert F.stats.factor_entries == plan.total_factor_entries
        rng = np.random.default_rng(seed + 100)
        b = rng.standard_normal(S.shape[0]) + 1j * rng.standard_normal(S.shape[0])
        x = np.concatenate(d.block_solve(F, split_blocks(b, K.sizes)))
        assert np.linalg.norm(S @ x - b) <= 1e-12 * np.linalg.norm(b)
        L, D = d.scatter_factor(F)
        p = _scalar_perm(plan)
        Sp = S[np.ix_(p, p)]
        assert np.linalg.norm(Sp - L @ D @ L.T) <= 1e-11 * np.linalg.norm(S)


def test_acceptance_criterion4_block_systems_vs_dense(cuda):
    """test_acceptance.py:100-119: 50 block systems (<= 12 blocks of <= 32)
    against the dense solve to 1e-11; pivots stay inside their blocks by
    construction (perm of each diagonal factor is a permutation of its block)."""
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import workloads as wl
    for seed in range(50):
        K, S = wl.rand_block_system(1000 + seed, max_blocks=12, max_size=32)
        F = d.block_ldlt(K, _plan(K))
        for j in range(F.plan.nblocks):
            assert sorted(F.diag[j].perm.tolist()) == list(range(int(F.plan.sizes_perm[j])))
        rng = np.random.default_rng(seed)
        b = rng.standard_normal(S.shape[0]) + 1j * rng.standard_normal(S.shape[0])
        x = np.concatenate(d.block_solve(F, split_blocks(b, K.sizes)))
        xd = np.linalg.solve(S, b)
        assert np.linalg.norm(x - xd) <= 1e-11 * np.linalg.norm(xd)


def test_arrow_matrix_vs_dense(cuda):
    """test_block_factor.py:35-51: block 0 coupled to every other block."""
    import paper_2002_05018_b200 as d
    rng = np.random.default_rng(35)
    sizes = [6, 4, 5, 3, 7]
    n = sum(sizes)
    off = np.concatenate([[0], np.cumsum(sizes)])
    S = np.zeros((n, n), dtype=complex)
    trip = []
    for i, si in enumerate(sizes):
        M = rand_complex_symmetric(si, 10 + i) + 2 * n * np.eye(si)
        S[off[i]:off[i + 1], off[i]:off[i + 1]] = M
        trip.append((i, i, M))
        if i:
            B = rng.standard_normal((si, sizes[0])) + 1j * rng.standard_normal((si, sizes[0]))
            S[off[i]:off[i + 1], :sizes[0]] = B
            S[:sizes[0], off[i]:off[i + 1]] = B.T
            trip.append((i, 0, B))
    K = d.from_blocks(sizes, trip)
    F = d.block_ldlt(K, _plan(K))
    b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    x = np.concatenate(d.block_solve(F, split_blocks(b, sizes)))
    xd = np.linalg.solve(S, b)
    assert np.linalg.norm(x - xd) <= 1e-11 * np.linalg.norm(xd)


@pytest.mark.parametrize("nsz,bad", [(8, 0), (256, 1), (300, 2)])
def test_singular_block_names_block_column(cuda, nsz, bad):
    """test_block_factor.py:144-149: a singular diagonal block raises
    SingularBlockError naming its block column -- on the exact (<= 128) and
    the cluster (256, 300) BK paths alike."""
    import paper_2002_05018_b200 as d
    sizes = [nsz] * 3
    trip = []
    for i in range(3):
        M = rand_complex_symmetric(nsz, 40 + i) + 3 * nsz * np.eye(nsz)
        if i == bad:
            M[:, 1] = 0.0
            M[1, :] = 0.0
        trip.append((i, i, M))
    for i in (1, 2):                 # coupling rows of the singular dof stay zero, so the
        C = 0.01 * np.ones((nsz, nsz), dtype=complex)   # Schur update keeps its row zero
        if i == bad:
            C[1, :] = 0.0
        trip.append((i, i - 1, C))
    K = d.from_blocks(sizes, trip)
    with pytest.raises(d.SingularBlockError, match=f"block column {bad}"):
        d.block_ldlt(K, _plan(K, d.identity_ordering(3)))


def test_tags_adjacency_and_reconstruction(cuda):
    """test_dense_factor.py:34-50, 145-158: every 2 is followed by 0 and
    reconstruction ||P M P^T - L D L^T|| <= 1e-13 ||M|| for indefinite
    matrices on every dense kernel size class."""
    import paper_2002_05018_b200 as d
    for n, seed in [(5, 1), (64, 2), (129, 3), (300, 4), (700, 5)]:
        M = rand_complex_symmetric(n, seed)
        M[np.diag_indices(n)] = 0.0            # forces 2x2 pivots
        f = d.dense_ldlt_bk(M)
        tags = f.tags
        two = np.flatnonzero(tags == 2)
        assert f.n_2x2 == two.size > 0
        assert np.all(two < n - 1) and np.all(tags[two + 1] == 0)
        assert set(np.unique(tags).tolist()) <= {0, 1, 2}
        assert np.count_nonzero(tags == 0) == two.size
        P = M[np.ix_(f.perm, f.perm)]
        assert np.linalg.norm(P - f.L @ f.dense_d() @ f.L.T) <= 1e-13 * n * np.linalg.norm(M)


def test_singular_large_subdomain_names_domain(cuda):
    """A rank-deficient subdomain on the batched panel path (n > 512) stops
    at its singular step and the error names the first bad domain in list
    order (subdomain.py:172-176)."""
    import paper_2002_05018_b200 as d
    rng = np.random.default_rng(8)
    n, m = 600, 8
    systems = []
    for b in range(3):
        G = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(2 * n)
        A = (G + G.T) / 2 + np.diag(rng.uniform(-1, 1, n))
        if b == 1:
            A[:, 123] = 0.0
            A[123, :] = 0.0
        D = np.zeros((n, m), dtype=complex)
        D[rng.choice(n, m, replace=False), np.arange(m)] = 1.0
        systems.append(d.SubdomainSystem(b, A, rng.standard_normal(n) + 0j, np.arange(n), [d.Coupling(0, D, 1)]))
    with pytest.raises(d.SingularDomainError, match="domain 1 is singular"):
        d.reduce_domains(systems)


def test_two_domain_sum_is_exact(cuda):
    """test_subdomain.py:188-198: the interface block assembled from two
    domains equals K_D1 + K_D2 exactly (one copy, one ordered add)."""
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import workloads as wl
    systems, part, *_ = wl.synthetic_d3m((2, 1, 1), 6, 4, 21)
    red = d.reduce_domains(systems)
    R = d.assemble_reduced(red, part)
    K1, K2 = np.asarray(red[0][0]), np.asarray(red[1][0])
    assert np.array_equal(np.asarray(R.K.blocks[(0, 0)]), K1 + K2)
    assert np.array_equal(np.asarray(R.g[0]), np.asarray(red[0][1]) + np.asarray(red[1][1]))

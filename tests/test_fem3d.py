"""3-D Nedelec front end checked on the CPU: the D3M path of
the oracle (restated reference algorithm) reproduces the monolithic sparse
solve (driver.run_verify's oracle, driver.py:145-155), the free-space problem
recovers the incident wave, and the lambda space has the expected sizes."""

from __future__ import annotations

import numpy as np
import pytest
import scipy.sparse.linalg as spla


def _oracle_d3m(model, oracle):
    from paper_2002_05018_b200 import fem3d
    from paper_2002_05018_b200.subdomain import interface_lambda_nodes
    systems = fem3d.subdomain_systems(model)
    kept = interface_lambda_nodes(model)
    red, facs = [], []
    for s in systems:
        K_D, g_d, fac = oracle.reduce_domain(s.A, np.concatenate([c.D for c in s.couplings], axis=1), s.f)
        red.append((K_D, g_d))
        facs.append(fac)
    sizes = [k.size for k in kept]
    blocks, g = oracle.assemble_reduced(red, [model.incident_interfaces(d) for d in range(model.n_domains)], sizes)
    adj = oracle.clique_adjacency(len(sizes), blocks.keys())
    plan = oracle.symbolic_factor(adj, oracle.reorder(adj, sizes), sizes)
    F = oracle.block_ldlt(blocks, plan)
    lam = oracle.block_solve(F, g)
    return oracle.recover_primal(facs, [s.f for s in systems], [[(c.interface, c.D) for c in s.couplings]
                                                                for s in systems], [s.dof_map for s in systems], lam)


@pytest.mark.parametrize("parts,radius", [((2, 1, 1), 0.0), ((2, 2, 1), 0.0), ((2, 2, 2), 0.15), ((1, 3, 2), 0.2)])
def test_d3m_equals_monolithic(oracle, parts, radius):
    from paper_2002_05018_b200 import fem3d
    model = fem3d.build_model(fem3d.FemProblem(4, 0.5, parts, sphere_radius=radius))
    A, f = fem3d.assemble_global(model)
    u = spla.spsolve(A.tocsc(), f[:, 0])
    sol = _oracle_d3m(model, oracle)
    assert np.linalg.norm(sol - u) / np.linalg.norm(u) <= 1e-10
    assert fem3d.global_residual(model, sol) <= 1e-11


def test_operator_symmetric_and_partition_exact():
    from paper_2002_05018_b200 import fem3d
    model = fem3d.build_model(fem3d.FemProblem(4, 0.5, (2, 2, 1)))
    A, f = fem3d.assemble_global(model)
    assert abs(A - A.T).max() == 0.0
    systems = fem3d.subdomain_systems(model)
    acc = np.zeros_like(f[:, 0])
    for s in systems:
        acc[s.dof_map] += s.f
        A = np.asarray(s.A)
        assert np.abs(A - A.T).max() <= 1e-14 * np.abs(A).max()
    assert np.abs(acc - f[:, 0]).max() <= 1e-15 * np.abs(f).max()


def test_free_space_recovers_incident_wave():
    from paper_2002_05018_b200 import fem3d
    errs = []
    for N in (4, 8):
        model = fem3d.build_model(fem3d.FemProblem(N, 0.5, (1, 1, 1)))
        A, f = fem3d.assemble_global(model)
        u = spla.spsolve(A.tocsc(), f[:, 0])
        ei = fem3d.interpolate_einc(model)
        errs.append(np.linalg.norm(u - ei) / np.linalg.norm(ei))
    assert errs[1] < 0.02 and errs[1] < errs[0] / 3      # ~h^2 convergence


def test_element_matrices_exact_properties():
    from paper_2002_05018_b200 import fem3d
    mesh = fem3d.build_cube_mesh(3, 1.0)
    S, M = fem3d.element_matrices(mesh)
    phi = lambda p: p[:, 0] ** 2 + p[:, 1] * p[:, 2]
    e = phi(mesh.nodes[mesh.edges[:, 1]]) - phi(mesh.nodes[mesh.edges[:, 0]])
    assert np.abs(np.einsum("tab,tb->ta", S, e[mesh.tet_edges])).max() <= 1e-13   # curl grad = 0
    assert np.allclose(M, np.transpose(M, (0, 2, 1)))


def test_configuration_sizes_and_lambda_space():
    """Exact unknown counts of BASELINE configs 1/2 and the lambda totals
    after the reference's cross-edge drop rule."""
    from paper_2002_05018_b200 import fem3d
    from paper_2002_05018_b200.subdomain import interface_lambda_nodes
    m1 = fem3d.build_model(fem3d.config1())
    assert m1.mesh.n_edges == 4184 and m1.n_domains == 2
    assert sum(k.size for k in interface_lambda_nodes(m1)) == 208
    mesh2 = fem3d.build_cube_mesh(16, 1.0)
    assert mesh2.n_edges == 31024
    m2 = fem3d.build_model(fem3d.config2())
    kept = interface_lambda_nodes(m2)
    total = sum(it.nodes.size for it in m2.interfaces)
    assert sum(k.size for k in kept) == 2448 and total - 2448 == 48
    sizes = np.bincount(m2.dom_of_tet)
    assert len(sizes) == 8


def test_sparse_subdomain_blocks_match_dense_assembly():
    """SparseBlock A_d / D_d (device-densified in reduce_domains) are the
    dense assembly bit for bit, signed zeros included."""
    from paper_2002_05018_b200 import fem3d
    model = fem3d.build_model(fem3d.FemProblem(4, 0.5, (2, 2, 1)))
    sp = fem3d.subdomain_systems(model, sparse=True)
    de = fem3d.subdomain_systems(model, sparse=False)
    bits = lambda a: np.asarray(a).view(np.uint64)
    for a, b in zip(sp, de):
        assert np.array_equal(bits(a.A), bits(b.A))
        assert np.array_equal(a.f, b.f)
        for ca, cb in zip(a.couplings, b.couplings):
            assert np.array_equal(bits(ca.D), bits(cb.D))


FEM_GOLDEN_CASES = [dict(cells=4, side=0.5, parts=(2, 2, 2), sphere_radius=0.15),
                    dict(cells=6, side=0.5, parts=(3, 1, 1), sphere_radius=0.2)]


@pytest.mark.parametrize("case", [0, 1])
def test_lambda_space_matches_reference_on_fem(case):
    """interface_lambda_nodes (subdomain.py:75-111) on the 3-D Nedelec
    partition equals the reference's own output (tools/gen_golden.py gen_fem)."""
    from conftest import golden
    from paper_2002_05018_b200 import fem3d, interface_lambda_nodes
    g = golden("fem_small.npz")
    model = fem3d.build_model(fem3d.FemProblem(**FEM_GOLDEN_CASES[case]))
    kept = interface_lambda_nodes(model)
    assert np.array_equal(np.concatenate(kept), g[f"c{case}_kept"])
    assert np.array_equal(np.array([k.size for k in kept]), g[f"c{case}_sizes"])

"""Generate tests/golden/*.npz by running the REFERENCE implementation.

Runs only in the build container, where /root/reference exists: it imports
the reference package ``ddsolve`` from /root/reference/pkg/src (numba JIT
backend, the reference's default, accel.py:33) and feeds it inputs from the
seeded generators of ``paper_2002_05018_b200.workloads`` (and the small random
generators below), recording its outputs.  The GPU box never reads
/root/reference: the tests compare against these committed fixtures.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tools/gen_golden.py [small|cfg4|cfg3|all]
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

from ddsolve import blockmat as rb, factor as rf, kernels as rk, ordering as ro  # noqa: E402
from ddsolve import subdomain as rs, symbolic as rsym  # noqa: E402

from paper_2002_05018_b200 import workloads as wl  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gen_golden_inputs import dense_suite, rand_sym  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gen_small():
    names, perms, tags, infos, n2, growth, scale, packed_digest = [], [], [], [], [], [], [], []
    full = {}
    for name, M in dense_suite():
        W = np.array(M, dtype=np.complex128, order="C")
        sc = np.abs(W).max()
        perm, tg, nn, gr, info = rk.bk_factor(W, 1e-12 * sc)
        names.append(name)
        perms.append(perm)
        tags.append(tg)
        infos.append(info)
        n2.append(nn)
        growth.append(gr)
        scale.append(sc)
        packed_digest.append(digest(np.tril(W)))
        if M.shape[0] <= 24 or name.startswith("big_256"):
            full[f"W_{name}"] = np.tril(W)
    np.savez_compressed(os.path.join(OUT, "dense_bk.npz"), names=np.array(names), info=np.array(infos),
                        n2x2=np.array(n2), growth=np.array(growth), scale=np.array(scale),
                        digest=np.array(packed_digest), perm=np.concatenate(perms), tags=np.concatenate(tags),
                        sizes=np.array([p.size for p in perms]), **full)

    # symbolic + ordering on random clique graphs (test_symbolic/test_ordering recipes)
    rng = np.random.default_rng(2024)
    recs = {}
    for c in range(60):
        n = int(rng.integers(1, 14))
        p = float(rng.uniform(0.05, 0.8))
        g = rb.CliqueGraph(n)
        for i in range(n):
            for j in range(i):
                if rng.random() < p:
                    g.add_edge(i, j)
        w = rng.integers(1, 9, size=n)
        order = ro.reorder(g, w)
        plan = rsym.symbolic_factor(g, order, w)
        nat = rsym.symbolic_factor(g, ro.identity_ordering(n), w)
        recs[f"g{c}_edges"] = np.array(g.edges(), dtype=np.int64).reshape(-1, 2)
        recs[f"g{c}_n"] = np.array(n)
        recs[f"g{c}_w"] = w
        recs[f"g{c}_perm"] = order.perm
        recs[f"g{c}_parent"] = plan.etree_parent
        recs[f"g{c}_pattern"] = np.concatenate([[len(x)] + list(x) for x in plan.pattern]).astype(np.int64)
        recs[f"g{c}_total"] = np.array(plan.total_factor_entries)
        recs[f"g{c}_nat_total"] = np.array(nat.total_factor_entries)
        recs[f"g{c}_fill"] = np.array(rsym.fill_blocks(plan, g), dtype=np.int64).reshape(-1, 2)
    np.savez_compressed(os.path.join(OUT, "planning.npz"), count=np.array(60), **recs)

    # block LDL^T on random block systems (conftest.py:26-60 generator)
    recs = {}
    for seed in range(30):
        K, S = wl.rand_block_system(seed, max_blocks=10, max_size=12, density=0.4)
        g = rb.clique_graph(K)
        order = ro.reorder(g, K.sizes)
        plan = rsym.symbolic_factor(g, order, K.sizes)
        F = rf.block_ldlt(rb.from_blocks(K.sizes, [(i, j, np.asarray(b)) for (i, j), b in K.blocks.items()]),
                          plan)
        rng2 = np.random.default_rng(900 + seed)
        b = rng2.standard_normal((S.shape[0], 3)) + 1j * rng2.standard_normal((S.shape[0], 3))
        off = np.concatenate([[0], np.cumsum(K.sizes)])
        x = np.concatenate(rf.block_solve(F, [b[off[i]:off[i + 1]] for i in range(K.nblocks)]))
        recs[f"s{seed}_order"] = order.perm
        recs[f"s{seed}_perm"] = np.concatenate([f.perm for f in F.diag])
        recs[f"s{seed}_tags"] = np.concatenate([f.tags for f in F.diag])
        recs[f"s{seed}_x"] = x
        recs[f"s{seed}_stats"] = np.array([F.stats.factor_entries, F.stats.flops, F.stats.peak_bytes,
                                           F.stats.n_2x2_pivots])
        recs[f"s{seed}_growth"] = np.array(F.stats.growth_factor)
    np.savez_compressed(os.path.join(OUT, "block_small.npz"), **recs)

    # DDM layer on the small synthetic D3M problem
    recs = {}
    for case, (grid, interior, fd, seed) in enumerate([((2, 2, 1), 12, 5, 0), ((3, 2, 2), 10, 4, 1)]):
        systems, part, n_glob = wl.synthetic_d3m(grid, interior, fd, seed)
        rsys_list = [rs.SubdomainSystem(s.domain, s.A, s.f, s.dof_map,
                                        [rs.Coupling(c.interface, c.D, c.sign) for c in s.couplings])
                     for s in systems]
        red = [rs.reduce_domain(s) for s in rsys_list]
        R = rs.assemble_reduced(red, part)
        g = rb.clique_graph(R.K)
        order = ro.reorder(g, R.K.sizes)
        plan = rsym.symbolic_factor(g, order, R.K.sizes)
        F = rf.block_ldlt(R.K, plan)
        lam = rf.block_solve(F, R.g)
        sol = rs.recover_primal(rsys_list, lam)
        for d, (KD, gd) in enumerate(red):
            recs[f"c{case}_KD{d}"] = KD
            recs[f"c{case}_gd{d}"] = gd
            recs[f"c{case}_fperm{d}"] = rsys_list[d].factor.perm
            recs[f"c{case}_ftags{d}"] = rsys_list[d].factor.tags
        recs[f"c{case}_lam"] = np.concatenate(lam)
        recs[f"c{case}_sol"] = sol
        recs[f"c{case}_order"] = order.perm
        recs[f"c{case}_kept"] = np.concatenate(rs.interface_lambda_nodes(part))
    np.savez_compressed(os.path.join(OUT, "ddm_small.npz"), **recs)
    print("small fixtures written")


def gen_fem():
    """The reference's own reduce_domain / assemble_reduced / block_ldlt /
    block_solve / recover_primal on small 3-D Nedelec models from fem3d.py
    (dense A_d, D_d handed over as numpy arrays; the FemModel serves as the
    partition shim: interfaces[*].{nodes, dom_lo, dom_hi}, incident_interfaces)."""
    from paper_2002_05018_b200 import fem3d
    recs = {}
    cases = [fem3d.FemProblem(4, 0.5, (2, 2, 2), sphere_radius=0.15),
             fem3d.FemProblem(6, 0.5, (3, 1, 1), sphere_radius=0.2)]
    for case, prob in enumerate(cases):
        model = fem3d.build_model(prob)
        systems = fem3d.subdomain_systems(model, rhs=0, sparse=False)
        rsys_list = [rs.SubdomainSystem(s.domain, np.asarray(s.A), np.asarray(s.f), s.dof_map,
                                        [rs.Coupling(c.interface, np.asarray(c.D), c.sign) for c in s.couplings])
                     for s in systems]
        t0 = time.perf_counter()
        red = [rs.reduce_domain(s) for s in rsys_list]
        R = rs.assemble_reduced(red, model)
        g = rb.clique_graph(R.K)
        order = ro.reorder(g, R.K.sizes)
        plan = rsym.symbolic_factor(g, order, R.K.sizes)
        F = rf.block_ldlt(R.K, plan)
        lam = rf.block_solve(F, R.g)
        sol = rs.recover_primal(rsys_list, lam)
        print(f"fem case {case}: n_sub {[s.n_dofs for s in systems]}, lambda {int(R.interface_sizes.sum())}, "
              f"{time.perf_counter() - t0:.1f}s")
        recs[f"c{case}_kept"] = np.concatenate(rs.interface_lambda_nodes(model))
        recs[f"c{case}_sizes"] = np.asarray(R.interface_sizes)
        for d in range(len(systems)):
            recs[f"c{case}_fperm{d}"] = rsys_list[d].factor.perm
            recs[f"c{case}_ftags{d}"] = rsys_list[d].factor.tags
            recs[f"c{case}_KD{d}"] = red[d][0]
        recs[f"c{case}_order"] = order.perm
        recs[f"c{case}_bperm"] = np.concatenate([f.perm for f in F.diag])
        recs[f"c{case}_lam"] = np.concatenate(lam)
        recs[f"c{case}_sol"] = sol
    np.savez_compressed(os.path.join(OUT, "fem_small.npz"), **recs)
    print("fem fixtures written")


def gen_cfg4():
    t0 = time.perf_counter()
    K = wl.config4_matrix()
    g = rb.clique_graph(K)
    plan = rsym.symbolic_factor(g, ro.identity_ordering(K.nblocks), K.sizes)
    Kr = rb.from_blocks(K.sizes, [(i, j, b) for (i, j), b in K.blocks.items()])
    F = rf.block_ldlt(Kr, plan)
    t1 = time.perf_counter()
    rhs = wl.config4_rhs(K)
    x = rf.block_solve(F, [b[:, :1] for b in rhs])
    t2 = time.perf_counter()
    np.savez_compressed(os.path.join(OUT, "cfg4.npz"),
                        perm=np.stack([f.perm for f in F.diag]).astype(np.int16),
                        tags=np.stack([f.tags for f in F.diag]),
                        n2x2=np.array([f.n_2x2 for f in F.diag]), growth=np.array([f.growth for f in F.diag]),
                        stats=np.array([F.stats.factor_entries, F.stats.flops, F.stats.peak_bytes,
                                        F.stats.n_2x2_pivots]),
                        x0=np.concatenate([xi[:, 0] for xi in x]),
                        pattern_total=np.array(plan.total_factor_entries),
                        t_factor=np.array(t1 - t0), t_solve1=np.array(t2 - t1))
    print(f"cfg4 reference: factor {t1 - t0:.1f}s, 1-RHS solve {t2 - t1:.1f}s, n2x2 {F.stats.n_2x2_pivots}")


def gen_cfg3(domains=(0, 1)):
    recs = {}
    for i in domains:
        A, D, f = wl.config3_domain(i)
        s = rs.SubdomainSystem(i, A, f, np.arange(A.shape[0]), [rs.Coupling(0, D, 1)])
        t0 = time.perf_counter()
        KD, gd = rs.reduce_domain(s)
        recs[f"perm{i}"] = s.factor.perm.astype(np.int16)
        recs[f"tags{i}"] = s.factor.tags
        recs[f"n2x2_{i}"] = np.array(s.factor.n_2x2)
        recs[f"growth{i}"] = np.array(s.factor.growth)
        recs[f"time{i}"] = np.array(time.perf_counter() - t0)
        if i == domains[0]:
            recs[f"KD{i}"] = KD
        recs[f"KDnorm{i}"] = np.array(np.linalg.norm(KD))
        print(f"cfg3 domain {i}: {time.perf_counter() - t0:.1f}s, n2x2 {s.factor.n_2x2}")
    np.savez_compressed(os.path.join(OUT, "cfg3.npz"), domains=np.array(domains), **recs)


def gen_blk():
    """A "D3M-BLK v1" dump written by the REFERENCE's save_blk (the golden-K
    exchange format, blockmat.py:132-146) of a small config-4-shaped K, and
    the reference's block_ldlt pivots / 1-RHS solution of the loaded K."""
    K = wl.config4_matrix(seed=21, grid=(2, 2, 3), n=12)
    Kr = rb.from_blocks(K.sizes, [(i, j, np.asarray(b)) for (i, j), b in K.blocks.items()])
    path = os.path.join(OUT, "k_small.blk")
    rb.save_blk(path, Kr)
    Kl = rb.load_blk(path)
    g = rb.clique_graph(Kl)
    order = ro.reorder(g, Kl.sizes)
    plan = rsym.symbolic_factor(g, order, Kl.sizes)
    F = rf.block_ldlt(Kl, plan)
    rng = np.random.default_rng(22)
    b = [rng.standard_normal(int(s)) + 1j * rng.standard_normal(int(s)) for s in Kl.sizes]
    x = rf.block_solve(F, b)
    np.savez_compressed(os.path.join(OUT, "k_small.npz"), order=order.perm,
                        perm=np.concatenate([f.perm for f in F.diag]), tags=np.concatenate([f.tags for f in F.diag]),
                        x=np.concatenate(x), b=np.concatenate(b))
    print("blk fixture written")


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    what = sys.argv[1] if len(sys.argv) > 1 else "small"
    if what in ("small", "all"):
        gen_small()
    if what in ("fem", "all"):
        gen_fem()
    if what in ("cfg4", "all"):
        gen_cfg4()
    if what in ("cfg3", "all"):
        gen_cfg3()
    if what in ("blk", "all"):
        gen_blk()

"""Generate the FEM-scale and full-RHS reference fixtures by running the
REFERENCE implementation (numba JIT backend) in the build container.

* ``fem_cfg1.npz`` / ``fem_cfg2.npz``: the reference's whole D3M pipeline
  (reduce_domain -> interface_lambda_nodes -> assemble_reduced -> reorder ->
  block_ldlt -> block_solve -> recover_primal) on BASELINE configs[0] and
  configs[1] exactly as ``fem3d.config1()`` / ``config2()`` build them (dense
  A_d and D_d handed to the reference; the FemModel is the partition shim).
  Subdomain reductions run in a process pool (they are independent,
  SPEC.md:176).  Stored: every subdomain's pivot sequence (perm, tags, n2x2),
  K_D (cfg1 full; cfg2 the first 64 rows plus the Frobenius norm), g_d, the
  reduced system's order and block pivots, lambda and the recovered field.
* ``cfg3_all.npz`` (``cfg3all``): the reference's reduce_domain on all 64
  config-3 subdomains: pivot sequences, K_D norms and first rows.
* ``cfg4_x16.npz``: the config-4 solution for all 16 RHS columns on a fixed
  row sample (rows 0..4095 and 2048 seeded random rows) plus column norms.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tools/gen_golden_femscale.py [cfg1|cfg2|cfg4|all|cfg3all]
"""

from __future__ import annotations

import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

OUT = os.path.join(ROOT, "tests", "golden")
CFG4_SAMPLE_SEED = 44


def cfg4_sample_rows(n: int) -> np.ndarray:
    rng = np.random.default_rng(CFG4_SAMPLE_SEED)
    extra = np.sort(rng.choice(np.arange(4096, n), 2048, replace=False))
    return np.concatenate([np.arange(4096), extra])


def _problem(name):
    from paper_2002_05018_b200 import fem3d
    return {"cfg1": fem3d.config1, "cfg2": fem3d.config2}[name]()


def _reduce_one(args):
    name, d = args
    from ddsolve import subdomain as rs
    from paper_2002_05018_b200 import fem3d
    model = fem3d.build_model(_problem(name))
    s = fem3d.subdomain_systems(model, rhs=0, sparse=False)[d]
    rsys = rs.SubdomainSystem(s.domain, np.asarray(s.A), np.asarray(s.f), s.dof_map,
                              [rs.Coupling(c.interface, np.asarray(c.D), c.sign) for c in s.couplings])
    t0 = time.perf_counter()
    KD, gd = rs.reduce_domain(rsys)
    dt = time.perf_counter() - t0
    print(f"{name} domain {d}: n={rsys.A.shape[0]} m={KD.shape[0]} {dt:.1f}s n2x2={rsys.factor.n_2x2}", flush=True)
    return d, KD, gd, rsys.factor, dt


def gen_fem(name: str, workers: int = 8):
    from ddsolve import blockmat as rb, factor as rf, ordering as ro, subdomain as rs, symbolic as rsym
    from paper_2002_05018_b200 import fem3d
    model = fem3d.build_model(_problem(name))
    systems = fem3d.subdomain_systems(model, rhs=0, sparse=False)
    nd = len(systems)
    t0 = time.perf_counter()
    with ProcessPoolExecutor(max_workers=min(workers, nd)) as ex:
        res = sorted(ex.map(_reduce_one, [(name, d) for d in range(nd)]), key=lambda r: r[0])
    t_red = time.perf_counter() - t0
    rsys_list = []
    for (d, KD, gd, fac, dt), s in zip(res, systems):
        rsys = rs.SubdomainSystem(s.domain, np.asarray(s.A), np.asarray(s.f), s.dof_map,
                                  [rs.Coupling(c.interface, np.asarray(c.D), c.sign) for c in s.couplings])
        rsys.factor = fac
        rsys_list.append(rsys)
    red = [(r[1], r[2]) for r in res]
    t1 = time.perf_counter()
    R = rs.assemble_reduced(red, model)
    g = rb.clique_graph(R.K)
    order = ro.reorder(g, R.K.sizes)
    plan = rsym.symbolic_factor(g, order, R.K.sizes)
    F = rf.block_ldlt(R.K, plan)
    lam = rf.block_solve(F, R.g)
    sol = rs.recover_primal(rsys_list, lam)
    t2 = time.perf_counter()
    recs = {"n_domains": np.array(nd), "t_reduce_wall": np.array(t_red), "t_rest": np.array(t2 - t1),
            "t_reduce_each": np.array([r[4] for r in res]), "workers": np.array(min(workers, nd))}
    recs["kept"] = np.concatenate(rs.interface_lambda_nodes(model))
    recs["sizes"] = np.asarray(R.interface_sizes)
    for d, KD, gd, fac, _ in res:
        recs[f"fperm{d}"] = fac.perm.astype(np.int16)
        recs[f"ftags{d}"] = fac.tags
        recs[f"fn2x2_{d}"] = np.array(fac.n_2x2)
        recs[f"fgrowth{d}"] = np.array(fac.growth)
        recs[f"KDnorm{d}"] = np.array(np.linalg.norm(KD))
        recs[f"KD{d}"] = KD if name == "cfg1" else KD[:64]
        recs[f"gd{d}"] = gd
    recs["order"] = order.perm
    recs["bperm"] = np.concatenate([f.perm for f in F.diag])
    recs["btags"] = np.concatenate([f.tags for f in F.diag])
    recs["lam"] = np.concatenate(lam)
    recs["sol"] = sol
    np.savez_compressed(os.path.join(OUT, f"fem_{name}.npz"), **recs)
    print(f"{name}: reduce {t_red:.1f}s wall ({nd} domains, {min(workers, nd)} procs), rest {t2 - t1:.1f}s, "
          f"lambda {int(R.interface_sizes.sum())}", flush=True)


def gen_cfg4_x16():
    from ddsolve import blockmat as rb, factor as rf, ordering as ro, symbolic as rsym
    from paper_2002_05018_b200 import workloads as wl
    os.environ["OPENBLAS_NUM_THREADS"] = str(os.cpu_count())
    t0 = time.perf_counter()
    K = wl.config4_matrix()
    g = rb.clique_graph(K)
    plan = rsym.symbolic_factor(g, ro.identity_ordering(K.nblocks), K.sizes)
    Kr = rb.from_blocks(K.sizes, [(i, j, b) for (i, j), b in K.blocks.items()])
    F = rf.block_ldlt(Kr, plan)
    t1 = time.perf_counter()
    rhs = wl.config4_rhs(K)
    x = np.concatenate(rf.block_solve(F, rhs))
    t2 = time.perf_counter()
    rows = cfg4_sample_rows(x.shape[0])
    np.savez_compressed(os.path.join(OUT, "cfg4_x16.npz"), rows=rows, x=x[rows], colnorm=np.linalg.norm(x, axis=0),
                        t_factor=np.array(t1 - t0), t_solve16=np.array(t2 - t1))
    print(f"cfg4 x16: factor {t1 - t0:.1f}s, 16-RHS solve {t2 - t1:.1f}s", flush=True)


def _cfg3_one(i):
    from ddsolve import subdomain as rs
    from paper_2002_05018_b200 import workloads as wl
    A, D, f = wl.config3_domain(i)
    s = rs.SubdomainSystem(i, A, f, np.arange(A.shape[0]), [rs.Coupling(0, D, 1)])
    t0 = time.perf_counter()
    KD, gd = rs.reduce_domain(s)
    dt = time.perf_counter() - t0
    print(f"cfg3 domain {i}: {dt:.1f}s n2x2 {s.factor.n_2x2}", flush=True)
    return (i, s.factor.perm.astype(np.int16), s.factor.tags, s.factor.n_2x2, s.factor.growth,
            float(np.linalg.norm(KD)), KD[:8].copy(), dt)


def gen_cfg3_all(workers: int = 8):
    """BASELINE configs[2]: the reference's reduce_domain on all 64
    subdomains (process pool): every pivot sequence, K_D norms and the first
    8 rows of every K_D (cfg3_all.npz; cfg3.npz keeps two full K_D)."""
    t0 = time.perf_counter()
    with ProcessPoolExecutor(max_workers=workers) as ex:
        res = sorted(ex.map(_cfg3_one, range(64)), key=lambda r: r[0])
    np.savez_compressed(os.path.join(OUT, "cfg3_all.npz"),
                        perm=np.stack([r[1] for r in res]), tags=np.stack([r[2] for r in res]),
                        n2x2=np.array([r[3] for r in res]), growth=np.array([r[4] for r in res]),
                        KDnorm=np.array([r[5] for r in res]), KDrows=np.stack([r[6] for r in res]),
                        t_each=np.array([r[7] for r in res]), t_wall=np.array(time.perf_counter() - t0))
    print(f"cfg3 all 64: {time.perf_counter() - t0:.1f}s wall", flush=True)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("cfg1", "all"):
        gen_fem("cfg1")
    if what in ("cfg2", "all"):
        gen_fem("cfg2")
    if what in ("cfg4", "all"):
        gen_cfg4_x16()
    if what == "cfg3all":
        gen_cfg3_all()

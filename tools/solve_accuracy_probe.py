"""Where does the unrefined config-4 residual come from?  (dev aid)

Factor config 4 on the GPU, then solve 2 RHS columns three ways and report
||Kx - b|| / ||b||:
  gpu       block_solve on the GPU (explicit Binv = L_jj^-1 P products)
  subst     the oracle's substitution solve (kernels.solve_unit_lower, as the
            reference) on the GPU factor's L / D / offdiag blocks
and the reference's own residual from tests/golden/cfg4_residuals.npz.
If `subst` is near the reference, the GPU solve's explicit inverses are the
cause; if not, the factor (panel TRSM through L^-1) is."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2002_05018_b200 as d
from oracle import d3m_oracle as O
from paper_2002_05018_b200 import workloads as wl

K = wl.config4_matrix()
plan = d.symbolic_factor(d.clique_graph(K), d.identity_ordering(K.nblocks), K.sizes)
rhs = [r[:, :2] for r in wl.config4_rhs(K)]
F = d.block_ldlt(K, plan)


def resid(x):
    Kx = [np.zeros_like(b) for b in rhs]
    for (i, j), blk in K.blocks.items():
        B = np.asarray(blk)
        Kx[i] += B @ x[j]
        if i != j:
            Kx[j] += B.T @ x[i]
    num = np.sqrt(sum(np.sum(np.abs(Kx[i] - rhs[i]) ** 2, axis=0) for i in range(K.nblocks)))
    den = np.sqrt(sum(np.sum(np.abs(rhs[i]) ** 2, axis=0) for i in range(K.nblocks)))
    return num / den


xg = [np.asarray(v) for v in d.block_solve(F, rhs)]
print("gpu   ", resid(xg))
diag = [O.OFactor(f.L, f.d, f.e, f.tags, f.perm, f.growth, f.n_2x2) for f in F.diag]
off = {k: np.asarray(v) for k, v in F.offdiag.items()}
OF = O.OBlockFactor({"sizes_perm": plan.sizes_perm, "pattern": plan.pattern, "perm": plan.order.perm}, diag, off)
xs = O.block_solve(OF, rhs)
print("subst ", resid(xs))
try:
    g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                             "cfg4_residuals.npz"))
    print("ref   ", g["residual"][:2])
except OSError:
    pass

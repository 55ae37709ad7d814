"""Reference residuals for config 4 (all 16 RHS) -> tests/golden/cfg4_residuals.npz.

Runs the REFERENCE block_ldlt / block_solve (numba JIT backend, build container
only; /root/reference is never read on the GPU box) on the seeded config-4
system and records, per RHS, ||K x - b|| / ||b|| of the reference's own
solution and its ||x||, so the GPU test can hold our residuals against the
reference's rather than against an absolute bound the reference itself does
not meet.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tools/gen_cfg4_residuals.py
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

from ddsolve import blockmat as rb, factor as rf, ordering as ro, symbolic as rsym  # noqa: E402

import bench  # noqa: E402
from paper_2002_05018_b200 import workloads as wl  # noqa: E402


def main():
    t0 = time.perf_counter()
    K = wl.config4_matrix()
    plan = rsym.symbolic_factor(rb.clique_graph(K), ro.identity_ordering(K.nblocks), K.sizes)
    Kr = rb.from_blocks(K.sizes, [(i, j, b) for (i, j), b in K.blocks.items()])
    F = rf.block_ldlt(Kr, plan)
    rhs = wl.config4_rhs(K)
    x = rf.block_solve(F, rhs)
    t1 = time.perf_counter()
    res = np.array([bench._residual(K, [b[:, c:c + 1] for b in rhs], [xi[:, c:c + 1] for xi in x])
                    for c in range(rhs[0].shape[1])])
    xn = np.sqrt(sum(np.sum(np.abs(xi) ** 2, axis=0) for xi in x))
    np.savez(os.path.join(ROOT, "tests", "golden", "cfg4_residuals.npz"), residual=res, xnorm=xn,
             seconds=np.array(t1 - t0))
    print("reference cfg4 residuals", res, "max", res.max(), f"({t1 - t0:.0f} s)")


if __name__ == "__main__":
    main()

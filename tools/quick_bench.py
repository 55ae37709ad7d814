"""Quick timing of the hot-path stages on the GPU (development aid)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2002_05018_b200 as d
from paper_2002_05018_b200 import workloads as wl

def cfg4():
    K = wl.config4_matrix()
    g = d.clique_graph(K); plan = d.symbolic_factor(g, d.identity_ordering(K.nblocks), K.sizes)
    rhs = wl.config4_rhs(K)
    for it in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        F = d.block_ldlt(K, plan)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        x = d.block_solve(F, rhs)
        torch.cuda.synchronize(); t2 = time.perf_counter()
        s = F._sched
        print(f"cfg4 it{it}: factor {t1-t0:.3f}s ({(s.flops_update+s.flops_trsm+s.flops_bk)/(t1-t0)/1e12:.2f} TF/s), solve16 {t2-t1:.3f}s, n2x2 {F.stats.n_2x2_pivots}", flush=True)
    S = K  # residual on a few blocks
    return F

def cfg3(count=8):
    systems = wl.config3_systems(count)
    for it in range(2):
        for s in systems: s.factor = None; s._d3m_D = None
        torch.cuda.synchronize(); t0 = time.perf_counter()
        red = d.reduce_domains(systems)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        print(f"cfg3 {count} domains it{it}: {t1-t0:.3f}s", flush=True)

if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("cfg4", "all"): cfg4()
    if what in ("cfg3", "all"): cfg3()

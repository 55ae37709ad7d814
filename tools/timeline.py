"""Headline step timeline from the per-launch CUDA-event intervals: how much
of the step has the update GEMMs running, only the critical chain, or
nothing (dev aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2002_05018_b200 as d
from paper_2002_05018_b200 import workloads as wl, _lib
from paper_2002_05018_b200.factor import to_device_blocks
from paper_2002_05018_b200.device import to_device, DeviceArray
K = wl.config4_matrix()
g = d.clique_graph(K)
plan = d.symbolic_factor(g, d.identity_ordering(K.nblocks), K.sizes)
Kd = to_device_blocks(K)
for it in range(2):
    _lib.counters_reset(timing=True)
    F = d.block_ldlt(Kd, plan)
    torch.cuda.synchronize()
    c = _lib.counters_read()
iv = _lib.timing_intervals()
t0, t1 = iv[:, 1].min(), iv[:, 2].max()
grid = np.linspace(t0, t1, 400001)
act = np.zeros((5, grid.size), dtype=bool)
for cls, a, b in iv:
    i0, i1 = np.searchsorted(grid, [a, b])
    act[int(cls), i0:i1] = True
dt = (t1 - t0) / (grid.size - 1)
gem = act[2]
crit = act[0] | act[1] | act[4]
print(f"factor span {t1 - t0:.1f} ms; union ms", {k: round(v, 1) for k, v in c["union_ms"].items()})
print(f"  gemm running: {gem.sum() * dt:.1f} ms; critical-only (no gemm): {(crit & ~gem).sum() * dt:.1f} ms;"
      f" idle: {(~gem & ~crit & ~act[3]).sum() * dt:.1f} ms")
print(f"  bk running w/o gemm: {(act[0] & ~gem).sum() * dt:.1f} ms; trsm w/o gemm: {(act[1] & ~gem).sum() * dt:.1f} ms;"
      f" misc w/o gemm: {(act[4] & ~gem & ~act[0] & ~act[1]).sum() * dt:.1f} ms")
# per decile of the factorisation
for q in range(10):
    s0, s1 = q * grid.size // 10, (q + 1) * grid.size // 10
    print(f"  decile {q}: gemm {gem[s0:s1].mean() * 100:.0f}%  crit-only {(crit & ~gem)[s0:s1].mean() * 100:.0f}%  "
          f"idle {(~gem & ~crit)[s0:s1].mean() * 100:.0f}%")

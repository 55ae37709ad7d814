"""Launch intervals of the last block columns of the config-4 factorisation
(dev aid): class, start, duration, gap to the previous launch's end."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2002_05018_b200 as d
from paper_2002_05018_b200 import workloads as wl, _lib
from paper_2002_05018_b200.factor import to_device_blocks
K = wl.config4_matrix()
plan = d.symbolic_factor(d.clique_graph(K), d.identity_ordering(K.nblocks), K.sizes)
Kd = to_device_blocks(K)
for it in range(2):
    _lib.counters_reset(timing=True)
    F = d.block_ldlt(Kd, plan)
    torch.cuda.synchronize()
    c = _lib.counters_read()
iv = _lib.timing_intervals()
t0 = iv[:, 1].min()
names = {0: "bk", 1: "trsm", 2: "gemm", 3: "solve", 4: "misc"}
n = int(sys.argv[1]) if len(sys.argv) > 1 else 70
print(f"{len(iv)} launches, span {iv[:, 2].max() - t0:.2f} ms")
for k in list(range(0, 24)) + list(range(len(iv) - n, len(iv))):
    c, a, b = iv[k]
    print(f"{k:5d} {names[int(c)]:5s} start {a - t0:8.3f} dur {1e3 * (b - a):8.1f} us")

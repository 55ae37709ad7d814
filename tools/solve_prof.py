"""cfg4 factor once, then the 16-RHS block solve inside an NVTX range (dev aid:
ncu --nvtx --nvtx-include 'solve/')."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2002_05018_b200 as d
from paper_2002_05018_b200 import workloads as wl, _lib
from paper_2002_05018_b200.device import to_device, DeviceArray
K = wl.config4_matrix()
from paper_2002_05018_b200.factor import to_device_blocks
Kd = to_device_blocks(K)
g = d.clique_graph(K)
plan = d.symbolic_factor(g, d.identity_ordering(K.nblocks), K.sizes)
F = d.block_ldlt(Kd, plan)
rhs = [DeviceArray(to_device(r)) for r in wl.config4_rhs(K)]
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    if it == 2:
        torch.cuda.nvtx.range_push("solve")
    x = d.block_solve(F, rhs)
    if it == 2:
        torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize(); print(f"solve {1e3*(time.perf_counter()-t0):.2f} ms", flush=True)

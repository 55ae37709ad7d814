"""Slow-mode frequency of the dataflow block solve (config 4, 16 RHS; dev aid).  Prints the kernel's own
CUDA-event time per pass."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2002_05018_b200 as d
from paper_2002_05018_b200 import _lib, workloads as wl
from paper_2002_05018_b200.factor import to_device_blocks
from paper_2002_05018_b200.device import DeviceArray, to_device
K = wl.config4_matrix()
plan = d.symbolic_factor(d.clique_graph(K), d.identity_ordering(K.nblocks), K.sizes)
F = d.block_ldlt(to_device_blocks(K), plan)
rhs = [DeviceArray(to_device(b)) for b in wl.config4_rhs(K)]
ts = []
for it in range(int(os.environ.get("ITERS", "26"))):
    _lib.counters_reset(timing=True)
    torch.cuda.synchronize()
    x = d.block_solve(F, rhs)
    torch.cuda.synchronize()
    c = _lib.counters_read(); _lib.counters_reset(False)
    ts.append(c["union_ms"].get("solve", 0.0))
ts = np.array(ts[2:])
print(f"{os.environ.get('TAG', '')}: " + " ".join(f"{v:.2f}" for v in ts) + f" | median {np.median(ts):.2f} min {ts.min():.2f} max {ts.max():.2f}", flush=True)

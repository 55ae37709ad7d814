"""Time block_solve alone on cfg4 (dev aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2002_05018_b200 as d
from paper_2002_05018_b200 import workloads as wl
from paper_2002_05018_b200.factor import to_device_blocks
from paper_2002_05018_b200.device import DeviceArray, to_device
K = wl.config4_matrix()
plan = d.symbolic_factor(d.clique_graph(K), d.identity_ordering(K.nblocks), K.sizes)
F = d.block_ldlt(to_device_blocks(K), plan)
rhs = [DeviceArray(to_device(b)) for b in wl.config4_rhs(K)]
for it in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x = d.block_solve(F, rhs)
    e1.record(); torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"solve {1e3*(t1-t0):.2f} ms wall, {e0.elapsed_time(e1):.2f} ms device", flush=True)

"""Per-stage timing of the cfg4 factor+solve with lookahead on/off (dev aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2002_05018_b200 as d
from paper_2002_05018_b200 import _lib, workloads as wl
from paper_2002_05018_b200.factor import to_device_blocks
from paper_2002_05018_b200.device import DeviceArray, to_device
K = wl.config4_matrix()
plan = d.symbolic_factor(d.clique_graph(K), d.identity_ordering(K.nblocks), K.sizes)
Kd = to_device_blocks(K)
rhs = [DeviceArray(to_device(b)) for b in wl.config4_rhs(K)]
mode = sys.argv[1] if len(sys.argv) > 1 else "both"
for la in ([False, True] if mode == "both" else [mode == "la"]):
    F = d.block_ldlt(Kd, plan, lookahead=la); x = d.block_solve(F, rhs); torch.cuda.synchronize()
    _lib.counters_reset(timing=True)
    t0 = time.perf_counter()
    F = d.block_ldlt(Kd, plan, lookahead=la); torch.cuda.synchronize()
    t1 = time.perf_counter()
    x = d.block_solve(F, rhs); torch.cuda.synchronize()
    t2 = time.perf_counter()
    c = _lib.counters_read(); _lib.counters_reset(False)
    print(f"lookahead={la}: factor {1e3*(t1-t0):.1f} ms, solve {1e3*(t2-t1):.1f} ms; per-class ms {{k: round(v,1) for k,v in c['ms'].items()}} n {c['n']}", flush=True)

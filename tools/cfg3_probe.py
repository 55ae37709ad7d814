"""Time the batched Schur reduction of config 3 (64 x n=2048, m=384) (dev aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2002_05018_b200 as d
from paper_2002_05018_b200 import _lib, workloads as wl
count = int(sys.argv[1]) if len(sys.argv) > 1 else 64
t0 = time.perf_counter()
systems = wl.config3_systems(count)
print(f"generated {count} domains in {time.perf_counter()-t0:.1f}s", flush=True)
for it in range(2):
    for s in systems: s.factor = None; s._d3m_D = None
    _lib.counters_reset(timing=True)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    red = d.reduce_domains(systems, keep=os.environ.get("KEEP", "factor"))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    c = _lib.counters_read(); _lib.counters_reset(False)
    print(f"cfg3 {count} domains: {1e3*(t1-t0):.1f} ms; per-class union ms " + str({k: round(v, 1) for k, v in c['union_ms'].items()}), flush=True)

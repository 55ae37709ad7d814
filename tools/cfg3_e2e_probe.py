"""Config-3 reduce end to end from host inputs (pinned tensors and numpy),
as bench.py's cfg3 e2e leg times it (dev aid)."""
import gc, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2002_05018_b200 as d
from paper_2002_05018_b200 import workloads as wl
host = wl.config3_systems(64)
pinned = [d.SubdomainSystem(s.domain, torch.from_numpy(s.A).pin_memory(),
                            torch.from_numpy(np.ascontiguousarray(s.f)).pin_memory(), s.dof_map,
                            [d.Coupling(c.interface, torch.from_numpy(np.ascontiguousarray(c.D)).pin_memory(),
                                        c.sign) for c in s.couplings]) for s in host]
for name, systems in (("pinned", pinned), ("numpy", host)):
    for it in range(3):
        for s in systems: s.factor = None; s._d3m_D = None
        gc.collect(); torch.cuda.synchronize(); t0 = time.perf_counter()
        red = d.reduce_domains(systems, keep="schur")
        outs = [(np.asarray(K_), np.asarray(g_)) for K_, g_ in red]
        torch.cuda.synchronize(); t1 = time.perf_counter()
        del red, outs
        print(f"cfg3 e2e {name}: {1e3*(t1-t0):.1f} ms", flush=True)

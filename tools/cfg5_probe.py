"""Config 5 (48^3 Nedelec, 4x4x4 subdomains, 4 RHS) through the full GPU D3M
pipeline (dev aid / DESIGN.md evidence)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2002_05018_b200 import fem3d, _lib

t0 = time.perf_counter()
model = fem3d.build_model(fem3d.config5())
t1 = time.perf_counter()
systems = fem3d.subdomain_systems(model, rhs=None)
t2 = time.perf_counter()
ns = sorted({s.n_dofs for s in systems})
print(f"edges={model.mesh.n_edges} domains={len(systems)} n_sub={ns} build={t1-t0:.1f}s systems={t2-t1:.1f}s",
      flush=True)
_lib.counters_reset(timing=True)
timers = {}
sol, systems, R, plan, F = fem3d.solve_d3m(model, rhs=None, keep=os.environ.get("KEEP", "auto"), timers=timers,
                                           systems=systems)
c = _lib.counters_read()
print("lambda", int(R.interface_sizes.sum()), "timers s", {k: round(v, 3) for k, v in timers.items()}, flush=True)
print("union ms", {k: round(v, 1) for k, v in c["union_ms"].items()}, "peak GB",
      round(torch.cuda.max_memory_allocated() / 1e9, 1), flush=True)
t3 = time.perf_counter()
res = fem3d.global_residual(model, sol, rhs=None)
print(f"residual={res:.3e} (check {time.perf_counter()-t3:.1f}s)", flush=True)

"""Time the D3M pipeline on the FEM configs (dev aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2002_05018_b200 import fem3d
for name in sys.argv[1:] or ["config1", "config2"]:
    t0 = time.perf_counter(); model = fem3d.build_model(getattr(fem3d, name)()); tb = time.perf_counter() - t0
    for it in range(2):
        tm = {}
        sol, systems, R, plan, F = fem3d.solve_d3m(model, timers=tm)
    res = fem3d.global_residual(model, sol)
    print(name, f"edges={model.mesh.n_edges} n_sub={systems[0].n_dofs} lambda={R.n_lambda} build={tb:.1f}s",
          {k: round(v * 1e3, 1) for k, v in tm.items()}, f"residual={res:.2e}", flush=True)

"""Config-2 reduce (8 x n=4184) timing with per-class device time (dev aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2002_05018_b200 import fem3d, subdomain, _lib
model = fem3d.build_model(fem3d.config2())
systems = fem3d.subdomain_systems(model)
for it in range(int(os.environ.get("REPS", "2"))):
    _lib.counters_reset(timing=True)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    red = subdomain.reduce_domains(systems)
    torch.cuda.synchronize()
    c = _lib.counters_read()
    print(f"reduce {1e3*(time.perf_counter()-t0):.1f} ms; union ms " +
          str({k: round(v, 1) for k, v in c["union_ms"].items()}), flush=True)

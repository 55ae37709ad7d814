"""One config-2 reduce (8 x n=4184) for profiling (dev aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2002_05018_b200 import fem3d, subdomain
model = fem3d.build_model(fem3d.config2())
systems = fem3d.subdomain_systems(model)
for it in range(int(os.environ.get("REPS", "2"))):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    red = subdomain.reduce_domains(systems)
    torch.cuda.synchronize(); print(f"reduce {1e3*(time.perf_counter()-t0):.1f} ms", flush=True)

"""Timeline of the config-3 reduce from pinned host inputs (torch.profiler
CUPTI trace: copies and kernels per stream), summarised (dev aid)."""
import gc, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2002_05018_b200 as d
from paper_2002_05018_b200 import workloads as wl
host = wl.config3_systems(64)
pinned = [d.SubdomainSystem(s.domain, torch.from_numpy(s.A).pin_memory(),
                            torch.from_numpy(np.ascontiguousarray(s.f)).pin_memory(), s.dof_map,
                            [d.Coupling(c.interface, torch.from_numpy(np.ascontiguousarray(c.D)).pin_memory(),
                                        c.sign) for c in s.couplings]) for s in host]
def run():
    for s in pinned: s.factor = None; s._d3m_D = None
    gc.collect(); torch.cuda.synchronize(); t0 = time.perf_counter()
    red = d.reduce_domains(pinned, keep="schur")
    outs = [(np.asarray(K_), np.asarray(g_)) for K_, g_ in red]
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t0)
for _ in range(4): print("warm", round(run(), 1), flush=True)
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    print("traced", round(run(), 1), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace("gpurun_out/cfg3_trace.json")
for _ in range(3): print("after", round(run(), 1), flush=True)

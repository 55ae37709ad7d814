"""Config-3 reduce: device-resident time vs batch chunk size, and pinned H2D
bandwidth (dev aid for the overlapped host-input path)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2002_05018_b200 as d
from paper_2002_05018_b200 import workloads as wl, subdomain as sd
from paper_2002_05018_b200.device import DeviceArray, to_device

n_gb = 1 << 30
h = torch.empty(n_gb, dtype=torch.uint8).pin_memory()
dv = torch.empty(n_gb, dtype=torch.uint8, device="cuda")
for _ in range(2): dv.copy_(h, non_blocking=True)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(4): dv.copy_(h, non_blocking=True)
torch.cuda.synchronize()
print(f"pinned H2D {4 * n_gb / (time.perf_counter() - t0) / 1e9:.1f} GB/s", flush=True)
del h, dv
host = wl.config3_systems(64)
dev = [d.SubdomainSystem(s.domain, DeviceArray(to_device(s.A)), DeviceArray(to_device(s.f)), s.dof_map,
                         [d.Coupling(c.interface, DeviceArray(to_device(c.D)), c.sign) for c in s.couplings])
       for s in host]
per = sd._domain_bytes(2048, 384, 1)
for chunk in [int(a) for a in (sys.argv[1:] or ["64", "32", "16", "8"])]:
    for it in range(3):
        for s in dev: s.factor = None; s._d3m_D = None
        torch.cuda.synchronize(); t0 = time.perf_counter()
        red = d.reduce_domains(dev, keep="schur", max_batch_bytes=per * chunk + 1)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        del red
    print(f"chunk {chunk}: {1e3*(t1-t0):.1f} ms for 64 domains", flush=True)

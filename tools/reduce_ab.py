"""Reduce-stage timing of configs 1, 2, 3 for A/B runs of libd3m builds or env switches (dev aid).
  [D3M_LIB=...] python tools/reduce_ab.py [cfg1] [cfg2] [cfg3]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2002_05018_b200 import fem3d, subdomain, _lib, workloads as wl
from paper_2002_05018_b200.device import DeviceArray, to_device
which = sys.argv[1:] or ["cfg1", "cfg2", "cfg3"]


def run(name, systems, keep):
    best = 1e9
    for it in range(4):
        for s in systems:
            s.factor = None
        _lib.counters_reset(timing=True)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        subdomain.reduce_domains(systems, keep=keep)
        torch.cuda.synchronize()
        best = min(best, 1e3 * (time.perf_counter() - t0))
        c = _lib.counters_read()
    print(f"{name}: reduce best {best:.1f} ms; last union ms " + str({k: round(v, 1) for k, v in c["union_ms"].items()}),
          flush=True)


if "cfg1" in which:
    run("cfg1", fem3d.subdomain_systems(fem3d.build_model(fem3d.config1())), "factor")
if "cfg2" in which:
    run("cfg2", fem3d.subdomain_systems(fem3d.build_model(fem3d.config2())), "factor")
if "cfg3" in which:
    systems = wl.config3_systems(64)
    for s in systems:
        s.A = DeviceArray(to_device(s.A))
    run("cfg3", systems, "schur")

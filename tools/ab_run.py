"""A/B timing of one libd3m build (select it with D3M_LIB): config-4 step
device-resident and from pinned host memory, and the config-2 FEM D3M (dev aid).

  D3M_LIB=paper_2002_05018_b200/libd3m_old.so python tools/ab_run.py [cfg4] [cfg2] [cfg3]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_2002_05018_b200 as d
from paper_2002_05018_b200 import _lib
from paper_2002_05018_b200.device import DeviceArray, to_device
from paper_2002_05018_b200.factor import to_device_blocks

what = sys.argv[1:] or ["cfg4", "cfg2"]
tag = os.path.basename(os.environ.get("D3M_LIB", "libd3m.so"))
out = {}
if "cfg4" in what:
    K, plan, rhs = bench._cfg4_host()
    Kd = to_device_blocks(K)
    rhs_d = [DeviceArray(to_device(b)) for b in rhs]
    for _ in range(2):
        F = d.block_ldlt(Kd, plan)
        x = d.block_solve(F, rhs_d)
    torch.cuda.synchronize()
    ts = []
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        F = d.block_ldlt(Kd, plan)
        x = d.block_solve(F, rhs_d)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out["cfg4_dev_ms"] = [round(t, 1) for t in ts]
    del F, x
    Kp, rhs_p = bench._pinned_inputs(K, rhs)
    ts = []
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        Fh = d.block_ldlt(Kp, plan)
        xh = [np.asarray(v) for v in d.block_solve(Fh, rhs_p)]
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
        del Fh, xh
    out["cfg4_e2e_ms"] = [round(t, 1) for t in ts]
    del Kd, Kp
if "cfg2" in what:
    r = bench._fem_secondary("cfg2", 3)
    out["cfg2"] = (r["d3m_ms"], r["stage_ms"])
if "cfg3" in what:
    r = bench._cfg3_secondary(3)
    out["cfg3"] = (r["ms_per_step"], r["e2e"]["ms_per_step"])
print(tag, out, flush=True)

"""Secondary-config timings in the bench's process context (after config-4 work) with per-class device time (dev aid)."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2002_05018_b200 as d
from paper_2002_05018_b200 import _lib, fem3d
from paper_2002_05018_b200.factor import to_device_blocks
from paper_2002_05018_b200.device import DeviceArray, to_device
peak = 37.1
if "nocfg4" not in sys.argv:
    K, plan, rhs = bench._cfg4_host()
    Kd = to_device_blocks(K)
    rhs_d = [DeviceArray(to_device(b)) for b in rhs]
    for _ in range(2):
        F = d.block_ldlt(Kd, plan); x = d.block_solve(F, rhs_d, refine=1)
    torch.cuda.synchronize()
    print("cfg4 done", flush=True)
if "nocfg3" not in sys.argv:
    print("cfg3", json.dumps({k: v for k, v in bench._cfg3_secondary(3, peak).items() if k in ("ms_per_step",)}), flush=True)
model = fem3d.build_model(fem3d.config1())
systems = fem3d.subdomain_systems(model, rhs=None)
for i in range(4):
    for s in systems:
        s.factor, s._d3m_D, s._d3m_X = None, None, None
    _lib.counters_reset(timing=True)
    timers = {}
    torch.cuda.synchronize(); t0 = time.perf_counter()
    sol, _, R, plan1, F1 = fem3d.solve_d3m(model, rhs=None, keep="auto", timers=timers, systems=systems, margins=(i == 0))
    torch.cuda.synchronize(); wall = time.perf_counter() - t0
    c = _lib.counters_read()
    print(f"cfg1 run {i}: wall {1e3*wall:.1f} ms reduce {1e3*timers['reduce']:.1f} ms; union ms",
          {k: round(v, 1) for k, v in c["union_ms"].items()}, "n", c["n"], flush=True)
    del F1

"""Secondary-config timings in the bench's process context (after config-4 work) (dev aid)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2002_05018_b200 as d
from paper_2002_05018_b200.factor import to_device_blocks
from paper_2002_05018_b200.device import DeviceArray, to_device
peak = 37.1
K, plan, rhs = bench._cfg4_host()
Kd = to_device_blocks(K)
rhs_d = [DeviceArray(to_device(b)) for b in rhs]
for _ in range(2):
    F = d.block_ldlt(Kd, plan); x = d.block_solve(F, rhs_d, refine=1)
torch.cuda.synchronize()
r3 = bench._cfg3_secondary(3, peak)
print("cfg3", r3["ms_per_step"], r3["samples_ms"], r3["e2e"]["ms_per_step"], flush=True)
for which in ("cfg1", "cfg2"):
    r = bench._fem_secondary(which, 4, peak)
    print(which, r["d3m_ms"], r["stage_ms"], flush=True)

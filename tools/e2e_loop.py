import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch, gc
import bench
import paper_2002_05018_b200 as d
from paper_2002_05018_b200.factor import to_device_blocks
from paper_2002_05018_b200.device import DeviceArray, to_device
K, plan, rhs = bench._cfg4_host()
Kd = to_device_blocks(K)
rhs_d = [DeviceArray(to_device(b)) for b in rhs]
for _ in range(3):
    F = d.block_ldlt(Kd, plan); x = d.block_solve(F, rhs_d, refine=1)
torch.cuda.synchronize()
del F, x
Kp, rhs_p = bench._pinned_inputs(K, rhs)
for it in range(10):
    t0 = time.perf_counter()
    Fh = d.block_ldlt(Kp, plan)
    t1 = time.perf_counter()
    xh = [np.asarray(v) for v in d.block_solve(Fh, rhs_p, refine=1)]
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    del Fh
    t3 = time.perf_counter()
    print(f"e2e {1e3*(t2-t0):.1f} ms (ldlt {1e3*(t1-t0):.1f}, solve {1e3*(t2-t1):.1f}); del {1e3*(t3-t2):.1f} ms; reserved {torch.cuda.memory_reserved()/1e9:.1f} GB", flush=True)

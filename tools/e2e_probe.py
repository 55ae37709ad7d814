"""Where the config-4 e2e step's extra time goes (dev aid): host time spent
inside block_ldlt / block_solve before they return, vs the device time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2002_05018_b200 as d
K, plan, rhs = bench._cfg4_host()
Kp, rhs_p = bench._pinned_inputs(K, rhs)
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    F = d.block_ldlt(Kp, plan)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    x = d.block_solve(F, rhs_p, refine=1)
    t3 = time.perf_counter()
    xh = [np.asarray(v) for v in x]
    t4 = time.perf_counter()
    print(f"ldlt host {1e3*(t1-t0):.1f} ms, ldlt total {1e3*(t2-t0):.1f}, solve {1e3*(t3-t2):.1f}, D2H {1e3*(t4-t3):.1f}, total {1e3*(t4-t0):.1f}", flush=True)
    del F

"""Host-side phases of the config-4 e2e block_ldlt call (dev aid): time to
first launch of the factorisation vs total."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2002_05018_b200 as d
from paper_2002_05018_b200 import factor as fac
K, plan, rhs = bench._cfg4_host()
Kp, rhs_p = bench._pinned_inputs(K, rhs)
orig_up = fac._upload_K_streamed
orig_call = fac._lib.call
stamps = {}
def up(*a, **k):
    t = time.perf_counter(); r = orig_up(*a, **k); stamps["upload_prep"] = time.perf_counter() - t; return r
def call(name, *a):
    if name == "d3m_block_ldlt_exec":
        stamps["exec_start"] = time.perf_counter()
    r = orig_call(name, *a)
    if name == "d3m_block_ldlt_exec":
        stamps["exec_return"] = time.perf_counter()
    return r
fac._upload_K_streamed = up
fac._lib.call = call
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    F = d.block_ldlt(Kp, plan)
    t1 = time.perf_counter()
    print(f"total {1e3*(t1-t0):.1f} ms; upload prep {1e3*stamps['upload_prep']:.1f}; exec call at +{1e3*(stamps['exec_start']-t0):.1f}, returns at +{1e3*(stamps['exec_return']-t0):.1f}", flush=True)
    del F

"""Critical-path analysis of the dataflow block solve on config 4 (dev aid):
D3M_FLOW_TRACE=1 stamps every work item (taken / inputs ready / done); this
prints per-type durations and the wait structure."""
import os, sys, ctypes
os.environ["D3M_FLOW_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2002_05018_b200 as d
from paper_2002_05018_b200 import _lib, workloads as wl, factor as fac
from paper_2002_05018_b200.factor import to_device_blocks
from paper_2002_05018_b200.device import DeviceArray, to_device
K = wl.config4_matrix()
plan = d.symbolic_factor(d.clique_graph(K), d.identity_ordering(K.nblocks), K.sizes)
F = d.block_ldlt(to_device_blocks(K), plan)
rhs = [DeviceArray(to_device(b)) for b in wl.config4_rhs(K)]
for _ in range(3):
    x = d.block_solve(F, rhs)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); x = d.block_solve(F, rhs); e1.record(); torch.cuda.synchronize()
print(f"solve {e0.elapsed_time(e1):.2f} ms")
items = fac.chain_split(fac.flow_items(F._sched.sizes, F._sched.pattern, F._sched.panel_rows)[0],
                        F._sched.sizes, F._sched.pattern)[0]
n = len(items)
buf = np.zeros(3 * n, dtype=np.int64)
lib = _lib.load()
lib.d3m_flow_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
m = lib.d3m_flow_trace(buf.ctypes.data, n)
tr = buf.reshape(-1, 3)[:m].astype(np.float64) / 1e3     # us
t0 = tr[:, 0].min()
tr -= t0
names = ["FA", "FD", "FB", "BC", "BR", "BE"]
print(f"span {tr[:, 2].max():.0f} us over {m} items")
for ty in range(6):
    sel = items[:m, 0] == ty
    if sel.any():
        run = tr[sel, 2] - tr[sel, 1]
        wait = tr[sel, 1] - tr[sel, 0]
        print(f"{names[ty]}: n={sel.sum():6d} run mean {run.mean():6.2f} us p50 {np.median(run):6.2f} p90 {np.percentile(run, 90):6.2f}"
              f"  wait mean {wait.mean():7.2f}")
# critical chain sample: FA of consecutive columns
fa = [(int(items[i, 1]), tr[i]) for i in range(m) if items[i, 0] == 0 and items[i, 2] == 0]
for (j, a), (j2, b) in list(zip(fa, fa[1:]))[60:66]:
    print(f"FA col {j}: ready {a[1]:9.1f} done {a[2]:9.1f}; next col ready after {b[1] - a[2]:6.2f} us")
be = [(int(items[i, 1]), tr[i]) for i in range(m) if items[i, 0] == 5 and items[i, 2] == 0]
for (j, a), (j2, b) in list(zip(be, be[1:]))[60:66]:
    print(f"BE col {j}: ready {a[1]:9.1f} done {a[2]:9.1f}; next col BE ready after {b[1] - a[2]:6.2f} us")

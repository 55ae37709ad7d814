"""Hand-off anatomy of the dataflow solve's forward/backward chain on config 4
(dev aid): for a few block columns, the taken / inputs-ready / done stamps of
the chain items (FA(j), FB(j -> parent rows), FA(j+1); BC/BR/BE backward)."""
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
items = fac.chain_split(fac.flow_items(F._sched.sizes, F._sched.pattern, F._sched.panel_rows)[0],
                        F._sched.sizes, F._sched.pattern)[0]
n = len(items)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
os.environ["D3M_FLOW_TRACE"] = "0"
buf = np.zeros(3 * n, dtype=np.int64)
lib = _lib.load()
lib.d3m_flow_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
m = lib.d3m_flow_trace(buf.ctypes.data, n)
tr = buf.reshape(-1, 3)[:m].astype(np.float64) / 1e3
tr -= tr[:, 0].min()
ty, jj, p0 = items[:m, 0], items[:m, 1], items[:m, 2]
names = ["FA", "FD", "FB", "BC", "BR", "BE"]
def show(sel, label):
    idx = np.nonzero(sel)[0]
    t = tr[idx]
    print(f"  {label:26s} n={len(idx):3d} q[{idx.min()}..{idx.max()}] taken {t[:,0].min():8.1f}..{t[:,0].max():8.1f}"
          f" ready {t[:,1].min():8.1f}..{t[:,1].max():8.1f} done {t[:,2].min():8.1f}..{t[:,2].max():8.1f}")
for j in (60, 61, 62):
    print(f"column {j}")
    show((ty == 0) & (jj == j), "FA(j)")
    show((ty == 1) & (jj == j), "FD(j)")
    show((ty == 2) & (jj == j) & (p0 < 256), "FB(j -> parent rows)")
    show((ty == 2) & (jj == j) & (p0 >= 256), "FB(j -> far rows)")
for j in (80, 79, 78):
    print(f"column {j} (backward)")
    show((ty == 3) & (jj == j) & (p0 == 0), "BC(j, chunk 0)")
    show((ty == 3) & (jj == j) & (p0 > 0), "BC(j, far chunks)")
    show((ty == 4) & (jj == j), "BR(j)")
    show((ty == 5) & (jj == j), "BE(j)")
# CTA occupancy: items running at time t
ev = np.concatenate([np.stack([tr[:, 0], np.ones(m)], 1), np.stack([tr[:, 2], -np.ones(m)], 1)])
ev = ev[np.argsort(ev[:, 0])]
busy = np.cumsum(ev[:, 1])
print(f"items in flight (taken, not done): mean {np.average(busy[:-1], weights=np.diff(ev[:, 0])):.0f}")
run = np.concatenate([np.stack([tr[:, 1], np.ones(m)], 1), np.stack([tr[:, 2], -np.ones(m)], 1)])
run = run[np.argsort(run[:, 0])]
rb = np.cumsum(run[:, 1])
print(f"items running (ready, not done): mean {np.average(rb[:-1], weights=np.diff(run[:, 0])):.0f}")
# producers of a consumer item's counters: which one finished last
deps = fac.flow_items(F._sched.sizes, F._sched.pattern, F._sched.panel_rows)[1]
prod = {}
for i in range(m):
    for c in (items[i, 6], items[i, 7]):
        if c >= 0:
            prod.setdefault(int(c), []).append(i)
def last_producers(i, k=4):
    out = []
    for dd in range(items[i, 5]):
        cnt, tgt = deps[items[i, 4] + dd]
        ps = sorted(prod.get(int(cnt), []), key=lambda q: tr[q, 2])
        out += [(tr[q, 2], names[ty[q]], int(jj[q]), int(p0[q]), int(items[q, 3]), int(cnt), int(tgt), len(ps)) for q in ps]
    out.sort(reverse=True)
    return out[:k]
for lab, sel in (("FA(61) tile 0", (ty == 0) & (jj == 61) & (p0 == 0)), ("FB(60->61) tile 0", (ty == 2) & (jj == 60) & (p0 == 0)),
                 ("BR(80) first", (ty == 4) & (jj == 80)), ("BC(80, chunk 0) tile 0", (ty == 3) & (jj == 80) & (p0 == 0))):
    i = int(np.nonzero(sel)[0][0])
    print(f"{lab}: taken {tr[i,0]:.1f} ready {tr[i,1]:.1f}; latest producers (done, type, j, p0, p1, counter, target, nprod):")
    for r in last_producers(i):
        print("   ", r)

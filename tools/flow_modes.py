"""The dataflow block solve in its fast and slow modes: what BR(j) waits for (dev aid; D3M_FLOW_TRACE stamps)."""
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
items, nchain = fac.chain_split(fac.flow_items(F._sched.sizes, F._sched.pattern, F._sched.panel_rows)[0],
                                F._sched.sizes, F._sched.pattern)[:2]
n = len(items)
print("items", n, "chain", nchain)
lib = _lib.load()
lib.d3m_flow_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
names = ["FA", "FD", "FB", "BC", "BR", "BE"]
seen = set()
J = int(os.environ.get("COL", "70"))
for it in range(12):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); x = d.block_solve(F, rhs); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    mode = "slow" if ms > 7.8 else "fast"
    if it < 2 or mode in seen:
        continue
    seen.add(mode)
    buf = np.zeros(3 * n, dtype=np.int64)
    m = lib.d3m_flow_trace(buf.ctypes.data, n)
    tr = buf.reshape(-1, 3)[:m].astype(np.float64) / 1e3     # us
    ty, col = items[:m, 0], items[:m, 1]
    be1 = [i for i in range(m) if ty[i] == 5 and col[i] == J + 1]
    t0 = max(tr[i, 2] for i in be1)
    print(f"== {mode} pass ({ms:.2f} ms); column {J} backward, times relative to the last BE({J + 1}) done")
    rows = []
    for i in range(m):
        if col[i] == J and ty[i] >= 3:
            rows.append((tr[i, 2] - t0, names[ty[i]], int(items[i, 2]), int(items[i, 3]), "chain" if i < nchain else "bulk",
                         tr[i, 0] - t0, tr[i, 1] - t0, i))
    rows.sort()
    bc = [r for r in rows if r[1] == "BC"]
    print(f"   BC items {len(bc)}; done before BE({J + 1}): {sum(r[0] < 0 for r in bc)}")
    for nm in ("BC", "BR", "BE"):
        rr = [r for r in rows if r[1] == nm and r[4] == "chain"]
        tk, rd, dn = np.array([r[5] for r in rr]), np.array([r[6] for r in rr]), np.array([r[0] for r in rr])
        print(f"   chain {nm}: {len(rr):3d} items; taken {tk.min():6.1f}..{tk.max():6.1f}  ready {rd.min():6.1f}..{rd.max():6.1f}"
              f"  done {dn.min():6.1f}..{dn.max():6.1f}  run mean {np.mean(dn - rd):5.1f} max {np.max(dn - rd):5.1f}")
    late = [r for r in rows if r[4] == "bulk" and r[0] > -5]
    print(f"   bulk items of the column finishing later than 5 us before BE({J + 1}): {len(late)}"
          + "".join(f" [{r[1]} ch {r[2]} ready {r[6]:.1f} done {r[0]:.1f}]" for r in late[-4:]))
    if len(seen) == 2:
        break

"""BK start times per block column of the config-4 factorisation (dev aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2002_05018_b200 as d
from paper_2002_05018_b200 import workloads as wl, _lib
from paper_2002_05018_b200.factor import to_device_blocks
K = wl.config4_matrix()
plan = d.symbolic_factor(d.clique_graph(K), d.identity_ordering(K.nblocks), K.sizes)
Kd = to_device_blocks(K)
for it in range(3):
    _lib.counters_reset(timing=True)
    F = d.block_ldlt(Kd, plan)
    torch.cuda.synchronize()
    c = _lib.counters_read()
iv = _lib.timing_intervals()
t0 = iv[:, 1].min()
bk = iv[iv[:, 0] == 0]
st = bk[:, 1] - t0
print("span", round(float(iv[:, 2].max() - t0), 2), "ms")
print("per-column BK start deltas (us), columns 0-19:", np.round(np.diff(st[:21]) * 1e3).astype(int).tolist())
print("columns 20-123 mean delta (us):", round(float(np.diff(st[20:124]).mean() * 1e3)))
print("columns 124-143 deltas (us):", np.round(np.diff(st[123:]) * 1e3).astype(int).tolist())
# chain elements per column (critical-stream launches in order: bk, tri_inv, trsm, dinv, next)
names = {0: "bk", 1: "trsm", 2: "gemm", 3: "solve", 4: "misc"}
bk_idx = np.flatnonzero(iv[:, 0] == 0)
for col in list(range(2, 20, 3)) + [60, 100, 130, 140]:
    a = bk_idx[col]
    b = bk_idx[col + 1] if col + 1 < len(bk_idx) else len(iv)
    seq = iv[a:b]
    parts = []
    prev_end = None
    for c_, s_, e_ in seq:
        gap = "" if prev_end is None else f"+{1e3 * (s_ - prev_end):.0f}"
        parts.append(f"{names[int(c_)]}{gap}:{1e3 * (e_ - s_):.0f}")
        if int(c_) != 2 or prev_end is None:
            prev_end = e_
    nxt = (iv[b, 1] - iv[a, 1]) * 1e3 if b < len(iv) else float("nan")
    print(f"col {col:3d} delta {nxt:6.0f} us | " + " ".join(parts))

"""Time the diagonal BK kernels on 256-wide config-4 blocks (dev aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2002_05018_b200 import _lib
from paper_2002_05018_b200.device import to_device, stream_ptr
from paper_2002_05018_b200 import workloads as wl
K = wl.config4_matrix()
blocks = [np.asarray(K.blocks[(j, j)]) for j in range(8)]
lib = _lib.load()
import ctypes
def run(kind, reps=3):
    ts = []
    for blk in blocks:
        W = to_device(blk).clone()
        n = blk.shape[0]
        perm = torch.empty(n, dtype=torch.int64, device="cuda"); tags = torch.empty(n, dtype=torch.int8, device="cuda")
        i32 = lambda: torch.empty(1, dtype=torch.int32, device="cuda"); f64 = lambda: torch.empty(1, dtype=torch.float64, device="cuda")
        n2, info, gr, sc, asy = i32(), i32(), f64(), f64(), f64()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        os.environ["D3M_DIAG_BK"] = "c" if kind == "cluster" else "b"
        fn = lib.d3m_bk_factor_batched if kind == "exact" else lib.d3m_bk_blocked_factor
        rc = fn(1, n, _lib.ptr(W), n*n, n, ctypes.c_double(1e-12), 1, _lib.ptr(perm), _lib.ptr(tags), _lib.ptr(n2), _lib.ptr(gr), _lib.ptr(info), _lib.ptr(sc), _lib.ptr(asy), None, stream_ptr())
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
        assert rc == 0
    return ts
for kind in (sys.argv[1:] or ["exact", "blocked", "cluster"]):
    run(kind)
    ts = run(kind)
    print(kind, "ms per 256-block:", [round(1e3*t, 3) for t in ts], flush=True)

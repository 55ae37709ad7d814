"""Cluster BK vs exact BK on one block: timing + first differing entry (dev aid)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2002_05018_b200 import _lib
from paper_2002_05018_b200.device import to_device, stream_ptr
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import rand_complex_symmetric
lib = _lib.load()

def fac(M, kind, cs=1):
    n = M.shape[0]
    W = to_device(M).clone()
    perm = torch.empty(n, dtype=torch.int64, device="cuda"); tags = torch.empty(n, dtype=torch.int8, device="cuda")
    i32 = lambda: torch.empty(1, dtype=torch.int32, device="cuda"); f64 = lambda: torch.empty(1, dtype=torch.float64, device="cuda")
    n2, info, gr, sc, asy = i32(), i32(), f64(), f64(), f64()
    os.environ["D3M_DIAG_BK"] = "cluster" if kind == "cluster" else "blocked"
    fn = lib.d3m_bk_factor_batched if kind == "exact" else lib.d3m_bk_blocked_factor
    torch.cuda.synchronize(); t0 = time.perf_counter()
    rc = fn(1, n, _lib.ptr(W), n * n, n, ctypes.c_double(1e-12), cs, _lib.ptr(perm), _lib.ptr(tags), _lib.ptr(n2),
            _lib.ptr(gr), _lib.ptr(info), _lib.ptr(sc), _lib.ptr(asy), None, stream_ptr())
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    assert rc == 0
    return np.tril(W.cpu().numpy()), perm.cpu().numpy(), tags.cpu().numpy(), gr.item(), dt

for n in (200, 256, 264, 320):
    M = rand_complex_symmetric(n, n)
    M[np.diag_indices(n)] += np.random.default_rng(n).uniform(-1, 1, n)
    We, pe, te, ge, _ = fac(M, "exact")
    for kind, cs in (("cluster", 1), ("cluster", 2), ("blocked", 1)):
        for _ in range(2):
            Wc, pc, tc, gc, dt = fac(M, kind, cs)
        kind = f"{kind}/cs{cs}"
        line = f"n={n} {kind}: {dt*1e3:.3f} ms perm_eq={np.array_equal(pe, pc)} tags_eq={np.array_equal(te, tc)} growth_eq={ge == gc}"
        if kind.startswith("cluster"):
            diff = np.argwhere(We != Wc)
            line += f" ndiff={len(diff)}"
            if len(diff):
                cols = diff[:, 1]
                j = cols.min()
                rows = diff[cols == j][:, 0]
                line += f" first col {j} rows {rows[:10].tolist()} tags[j-2:j+2]={te[max(0,j-2):j+2].tolist()} n2x2={int((te==2).sum())}"
                line += f" diffcols={np.unique(cols)[:12].tolist()}"
        print(line, flush=True)

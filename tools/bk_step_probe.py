"""Per-step cost of the diagonal BK kernels (dev aid): the single-CTA exact
kernel (global memory) and the cluster kernel (shared memory, CS CTAs) on one
dense block of order n, timed with CUDA events over repeated launches."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2002_05018_b200 import _lib
from paper_2002_05018_b200.device import stream_ptr

lib = _lib.load()
P = _lib.ctypes.c_void_p


def timed(n, cs, reps=20):
    rng = np.random.default_rng(n)
    G = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(2 * n)
    M = (G + G.T) / 2
    M[np.diag_indices(n)] += rng.uniform(-2, 2, n)
    W0 = torch.from_numpy(M).cuda()
    W = W0.clone()
    perm = torch.empty(n, dtype=torch.int64, device="cuda")
    tags = torch.empty(n, dtype=torch.int8, device="cuda")
    i32 = [torch.empty(1, dtype=torch.int32, device="cuda") for _ in range(2)]
    f64 = [torch.empty(1, dtype=torch.float64, device="cuda") for _ in range(3)]
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    def run():
        W.copy_(W0)
        if cs == 0:
            rc = lib.d3m_bk_factor_batched(1, n, P(W.data_ptr()), n * n, n, 1e-12, 1, P(perm.data_ptr()),
                                           P(tags.data_ptr()), P(i32[0].data_ptr()), P(f64[0].data_ptr()),
                                           P(i32[1].data_ptr()), P(f64[1].data_ptr()), P(f64[2].data_ptr()), None,
                                           None, stream_ptr())
            assert rc == 0
        else:
            os.environ["D3M_BKC_CS"] = str(cs)
            import paper_2002_05018_b200 as d
            raise SystemExit("cluster path: use block_ldlt")
    if cs == 0:
        run(); torch.cuda.synchronize()
        e0.record(s)
        for _ in range(reps):
            run()
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    import paper_2002_05018_b200 as d
    os.environ["D3M_BKC_CS"] = str(cs)
    K = d.from_blocks([n], [(0, 0, M)])
    plan = d.symbolic_factor(d.clique_graph(K), d.identity_ordering(1), K.sizes)
    _lib.counters_reset(timing=True)
    for _ in range(reps):
        d.block_ldlt(K, plan)
    torch.cuda.synchronize()
    c = _lib.counters_read()
    _lib.counters_reset(timing=False)
    return c["ms"]["bk"] / c["n"]["bk"]


for n in (() if os.environ.get("NO_EXACT") else (32, 64, 96, 128)):
    ms = timed(n, 0)
    print(f"exact  n={n:4d}: {ms * 1e3:8.1f} us  {ms * 1e3 / n:6.2f} us/step", flush=True)
for cs in tuple(int(c) for c in os.environ.get("CS_LIST", "8,4").split(",")):
    for n in (130, 192, 256):
        ms = timed(n, cs)
        print(f"cluster{cs} n={n:4d}: {ms * 1e3:8.1f} us  {ms * 1e3 / n:6.2f} us/step", flush=True)

"""Standalone throughput of the TMA-staged update GEMM against the cp.async half-tile kernel (dev aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2002_05018_b200 import _lib
from paper_2002_05018_b200.device import stream_ptr
M = N = 6144
P = _lib.ptr
for K in (256, 448, 1024):
    A = torch.randn(M, K, dtype=torch.complex128, device="cuda")
    B = torch.randn(N, K, dtype=torch.complex128, device="cuda")
    C = torch.randn(M, N, dtype=torch.complex128, device="cuda")
    d_tasks = torch.empty(64, dtype=torch.uint8, device="cuda")

    def task():
        t = np.zeros(1, dtype=_lib.GEMM_TASK)
        t["m"], t["n"], t["k"], t["lda"], t["ldb"], t["ldc"], t["flags"] = M, N, K, K, K, N, _lib.GEMM_SUB
        return t
    runs = {"cp.async": lambda: _lib.call("d3m_zgemm_grouped", 0, 0, P(A), P(B), P(C), _lib.hptr(task()), 1, P(d_tasks), stream_ptr()),
            "tma": lambda: _lib.call("d3m_zgemm_tma_panels", P(A), M, P(B), N, K, P(C), _lib.hptr(task()), 1, P(d_tasks), stream_ptr())}
    for name, fn in runs.items():
        best = 1e9
        for rep in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            fn(); torch.cuda.synchronize()
            e0.record()
            for _ in range(5):
                fn()
            e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / 5)
        print(f"K={K} {name:9s}: {best:.3f} ms, {8 * M * N * K / best / 1e9:.2f} TFLOP/s (incl. task upload / map encode)", flush=True)

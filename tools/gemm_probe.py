"""Standalone throughput of the grouped DMMA GEMM (C -= A B^T, 64x64 tiles) (dev aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2002_05018_b200 import _lib
from paper_2002_05018_b200.device import stream_ptr
M = N = 6144; K = int(os.environ.get("K", "256"))
A = torch.randn(M, K, dtype=torch.complex128, device="cuda")
B = torch.randn(N, K, dtype=torch.complex128, device="cuda")
C = torch.randn(M, N, dtype=torch.complex128, device="cuda")
t = np.zeros(1, dtype=_lib.GEMM_TASK)
t["m"], t["n"], t["k"], t["lda"], t["ldb"], t["ldc"], t["flags"] = M, N, K, K, K, N, _lib.GEMM_SUB
d_tasks = torch.empty(64, dtype=torch.uint8, device="cuda")
P = _lib.ptr
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        _lib.call("d3m_zgemm_grouped", 0, 0, P(A), P(B), P(C), _lib.hptr(t), 1, P(d_tasks), stream_ptr())
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"K={K}: {ms:.3f} ms, {8 * M * N * K / ms / 1e9:.2f} TFLOP/s", flush=True)

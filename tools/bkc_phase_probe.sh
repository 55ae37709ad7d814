#!/bin/bash
# Build a profiling variant of the cluster BK and print per-phase cycles of CTA 0 (dev aid)
set -e
cd "$(dirname "$0")/.."
D=/tmp/bkcprof; mkdir -p $D
SRCS=$(python -c "import sys; sys.path.insert(0, 'paper_2002_05018_b200'); import build_ext; print(' '.join(f[:-3] for f in build_ext.SOURCES))")
for f in $SRCS; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -DD3M_BK_PROFILE --expt-relaxed-constexpr \
    -I paper_2002_05018_b200/csrc -I include -c paper_2002_05018_b200/csrc/$f.cu -o $D/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/libd3m.so $D/*.o -lcudart
python - <<'PY'
import ctypes, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2002_05018_b200 import _lib, workloads as wl
_lib.LIB_PATH = "/tmp/bkcprof/libd3m.so"
lib = _lib.load()
from paper_2002_05018_b200.device import to_device, stream_ptr
os.environ["D3M_DIAG_BK"] = "cluster"
K = wl.config4_matrix()
for j in range(4):
    blk = np.asarray(K.blocks[(j, j)]); n = blk.shape[0]
    W = to_device(blk).clone()
    perm = torch.empty(n, dtype=torch.int64, device="cuda"); tags = torch.empty(n, dtype=torch.int8, device="cuda")
    z = lambda t: torch.zeros(1, dtype=t, device="cuda")
    scr = torch.zeros(32, dtype=torch.float64, device="cuda")
    rc = lib.d3m_bk_blocked_factor(1, n, _lib.ptr(W), n*n, n, ctypes.c_double(1e-12), 1, _lib.ptr(perm), _lib.ptr(tags),
        _lib.ptr(z(torch.int32)), _lib.ptr(z(torch.float64)), _lib.ptr(z(torch.int32)), _lib.ptr(z(torch.float64)), _lib.ptr(z(torch.float64)), _lib.ptr(scr), stream_ptr())
    torch.cuda.synchronize()
    p = scr.cpu().numpy()
    pn = ["wait", "merge", "decide+rowmax+swap", "arrive", "l0", "col-update+push+hypot", "argmax+post"]
    bn = ["wait", "merge", "refill+mult+arrive", "bulk"]
    print("pivot warp:", " ".join(f"{nm}={v/1e3:.0f}K" for nm, v in zip(pn, p[:7])), f"total={p[:8].sum()/1e6:.2f}M cycles")
    print("bulk warps:", " ".join(f"{nm}={v/1e3:.0f}K" for nm, v in zip(bn, p[8:12])), f"total={p[8:16].sum()/1e6:.2f}M cycles")
    print(f"CTA 0: prologue {p[16]/1e3:.0f}K, step loop {p[17]/1e3:.0f}K, write-back {p[18]/1e3:.0f}K cycles")
PY

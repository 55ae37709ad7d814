#!/bin/bash
# Per-phase clocks of the cluster BK (CTA 0's pivot warp and first bulk thread)
# from a -DD3M_BK_PROFILE build of libd3m (dev aid; run under gpurun).
set -e
cd "$(dirname "$0")/.."
D=/tmp/bkcprof; mkdir -p $D
if [ -z "$SKIP_BUILD" ]; then
SRCS=$(python -c "import sys; sys.path.insert(0, 'paper_2002_05018_b200'); import build_ext; print(' '.join(build_ext.SOURCES))")
for f in $SRCS; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -DD3M_BK_PROFILE --expt-relaxed-constexpr \
    -I paper_2002_05018_b200/csrc -I include -c paper_2002_05018_b200/csrc/$f -o $D/${f%.*}.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/libd3m.so $D/*.o -lcudart
fi
D3M_LIB=${D3M_LIB:-$D/libd3m.so} python - <<'PY'
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2002_05018_b200 as d
from paper_2002_05018_b200 import _lib, workloads as wl
lib = _lib.load()
K = wl.config4_matrix()
for cs in (os.environ.get("CS_LIST", "8,4").split(",")):
    os.environ["D3M_BKC_CS"] = cs
    for j in range(2):
        blk = np.asarray(K.blocks[(j, j)])
        Kj = d.from_blocks([256], [(0, 0, blk)])
        plan = d.symbolic_factor(d.clique_graph(Kj), d.identity_ordering(1), Kj.sizes)
        d.block_ldlt(Kj, plan, lookahead=False)
        torch.cuda.synchronize()
        p = np.zeros(32)
        lib.d3m_bkc_prof_read(p.ctypes.data_as(ctypes.c_void_p))
        pn = ["wait", "merge", "3P-swap+arrive", "decide", "l0", "col-update+push+hypot", "argmax+post", "up"]
        bn = ["wait", "merge", "refill+mult+arrive", "bulk"]
        print(f"CS={cs} block {j}: pivot warp:", " ".join(f"{nm}={v/1e3:.0f}K" for nm, v in zip(pn, p[:8])),
              f"total={p[:8].sum()/1e6:.3f}M cycles")
        print(f"CS={cs} block {j}: bulk warps:", " ".join(f"{nm}={v/1e3:.0f}K" for nm, v in zip(bn, p[8:12])),
              f"total={p[8:16].sum()/1e6:.3f}M")
        print(f"CS={cs} block {j}: CTA 0: prologue {p[16]/1e3:.0f}K, step loop {p[17]/1e3:.0f}K, "
              f"write-back {p[18]/1e3:.0f}K cycles; steps {p[22]:.0f}: rowmax {p[19]:.0f}, interchange {p[20]:.0f}, "
              f"2x2 {p[21]:.0f}; decide phase: plain steps {(p[2]+p[3])/max(1, p[22]-p[19]):.0f}, rowmax steps {p[23]/max(1, p[19]):.0f} cycles/step", flush=True)
PY

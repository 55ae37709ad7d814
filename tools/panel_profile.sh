#!/bin/bash
# Per-phase clocks of the subdomain panel BK (matrix 0, rank-0 CTA, thread 0) from a
# -DD3M_PANEL_PROFILE build of libd3m (dev aid; run under gpurun).  CFGS="cfg1 cfg2 cfg3"
set -e
cd "$(dirname "$0")/.."
D=/tmp/panelprof; mkdir -p $D
SRCS=$(python -c "import sys; sys.path.insert(0, 'paper_2002_05018_b200'); import build_ext; print(' '.join(build_ext.SOURCES))")
for f in $SRCS; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -DD3M_PANEL_PROFILE --expt-relaxed-constexpr \
    -I paper_2002_05018_b200/csrc -I include -c paper_2002_05018_b200/csrc/$f -o $D/${f%.*}.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/libd3m.so $D/*.o -lcudart
D3M_LIB=$D/libd3m.so python - <<'PY'
import ctypes, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2002_05018_b200 import fem3d, subdomain, _lib, workloads as wl
from paper_2002_05018_b200.device import DeviceArray, to_device
lib = _lib.load()
names = ["gemv(k)", "argmax(k)", "merge(k)", "gemv(imax)", "argmax+merge(imax)", "interchange", "L store", "loop top"]
def run(name, systems, keep):
    for it in range(2):
        for s in systems:
            s.factor = None
        out = (ctypes.c_double * 16)()
        lib.d3m_panel_prof_read(out, 1)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        subdomain.reduce_domains(systems, keep=keep)
        torch.cuda.synchronize(); ms = 1e3 * (time.perf_counter() - t0)
        lib.d3m_panel_prof_read(out, 0)
    v = list(out)
    steps = max(v[8], 1.0)
    tot = sum(v[:8])
    print(f"{name}: reduce {ms:.1f} ms; {int(v[8])} steps, {int(v[9])} rowmax steps, {int(v[10])} interchanges; "
          f"{tot / steps:.0f} cycles per step ({tot / steps / 1.965e3:.2f} us)")
    for i, nm in enumerate(names):
        print(f"   {nm:20s} {v[i] / steps:8.0f} cycles per step ({100 * v[i] / tot:4.1f}%)")
for c in os.environ.get("CFGS", "cfg1 cfg2 cfg3").split():
    if c == "cfg1":
        run(c, fem3d.subdomain_systems(fem3d.build_model(fem3d.config1())), "factor")
    if c == "cfg2":
        run(c, fem3d.subdomain_systems(fem3d.build_model(fem3d.config2())), "factor")
    if c == "cfg3":
        systems = wl.config3_systems(64)
        for s in systems:
            s.A = DeviceArray(to_device(s.A))
        run(c, systems, "schur")
PY

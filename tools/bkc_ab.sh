#!/bin/bash
# A/B of cluster-BK compile-time variants (dev aid; run under gpurun):
#   VARIANTS="base:|late:-DD3M_BKC_LATE_ARRIVE" bash tools/bkc_ab.sh
# builds libd3m per variant (and its -DD3M_BK_PROFILE twin) under /tmp and
# runs tools/bk_step_probe.py (CS_LIST) and the phase profile for each.
set -e
cd "$(dirname "$0")/.."
SRCS=$(python -c "import sys; sys.path.insert(0, 'paper_2002_05018_b200'); import build_ext; print(' '.join(build_ext.SOURCES))")
IFS='|' read -ra VS <<< "${VARIANTS:-base:}"
for v in "${VS[@]}"; do
  name=${v%%:*}; flags=${v#*:}
  for prof in 0 1; do
    D=/tmp/bkab_${name}_$prof; mkdir -p $D
    pf=""; [ $prof = 1 ] && pf="-DD3M_BK_PROFILE"
    for f in $SRCS; do
      nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC $flags $pf --expt-relaxed-constexpr \
        -I paper_2002_05018_b200/csrc -I include -c paper_2002_05018_b200/csrc/$f -o $D/${f%.*}.o &
    done
    wait
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/libd3m.so $D/*.o -lcudart
  done
done
for v in "${VS[@]}"; do
  name=${v%%:*}
  echo "== variant $name"
  NO_EXACT=1 D3M_LIB=/tmp/bkab_${name}_0/libd3m.so timeout 300 python tools/bk_step_probe.py
  D3M_LIB=/tmp/bkab_${name}_1/libd3m.so SKIP_BUILD=1 CS_LIST=${PROF_CS:-8} bash tools/bkc_profile.sh | grep -v "^$"
done

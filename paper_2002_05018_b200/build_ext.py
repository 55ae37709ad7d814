"""Build libd3m.so in-tree with nvcc for sm_100a (called by __graft_entry__.build)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
OUT = os.path.join(HERE, "libd3m.so")
SOURCES = ["bk_exact.cu", "bk_cluster.cu", "zgemm_dmma.cu", "ldlt_solve.cu", "skinny_dmma.cu", "bk_panel.cu", "solve_blocked.cu", "d3m_misc.cu", "d3m_capi.cu", "d3m_plan.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"]


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(INCLUDE, "d3m.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return OUT
    nvcc = os.environ.get("NVCC", "nvcc")
    objdir = os.path.join(HERE, "_obj")
    os.makedirs(objdir, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if not f.endswith((".cu", ".cpp"))]
    headers.append(os.path.join(INCLUDE, "d3m.h"))
    hdr_t = max(os.path.getmtime(h) for h in headers)
    objs, cmds = [], []
    for src in SOURCES:
        obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
        objs.append(obj)
        srcp = os.path.join(CSRC, src)
        if not force and os.path.exists(obj) and os.path.getmtime(obj) > max(hdr_t, os.path.getmtime(srcp)):
            continue
        cmds.append([nvcc, *ARCH, *FLAGS, "-I", CSRC, "-I", INCLUDE, "-c", srcp, "-o", obj])
    # objects compile independently: run the nvcc invocations in parallel
    procs = []
    for cmd in cmds:
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((cmd, subprocess.Popen(cmd)))
    bad = [cmd for cmd, pr in procs if pr.wait() != 0]
    if bad:
        raise subprocess.CalledProcessError(1, bad[0])
    tmp = OUT + ".tmp"
    subprocess.check_call([nvcc, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"])
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))

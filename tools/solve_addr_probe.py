"""Which SMs took the chain role in the dataflow block solve, against the pass time (dev aid).
The kernel has two time modes on config 4 (5.97 / 7.55 ms per 16-RHS pass)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2002_05018_b200 as d
from paper_2002_05018_b200 import _lib, workloads as wl
from paper_2002_05018_b200.factor import to_device_blocks
from paper_2002_05018_b200.device import DeviceArray, to_device
K = wl.config4_matrix()
plan = d.symbolic_factor(d.clique_graph(K), d.identity_ordering(K.nblocks), K.sizes)
F = d.block_ldlt(to_device_blocks(K), plan)
rhs = [DeviceArray(to_device(b)) for b in wl.config4_rhs(K)]
cap = {}
orig = _lib.call


def hook(name, *args):
    if name == "d3m_block_solve_dataflow":
        cap["cnt"], cap["n"] = args[7].value, int(args[8])
        cap["ptrs"] = [a.value for a in args if isinstance(a, ctypes.c_void_p)]
    return orig(name, *args)


_lib.call = hook
import paper_2002_05018_b200.factor as fmod
fmod._lib.call = hook
rt = ctypes.CDLL("libcudart.so.12")
EX = _lib.FLOW_EXTRA_COUNTERS
for it in range(int(os.environ.get("ITERS", "24"))):
    _lib.counters_reset(timing=True)
    torch.cuda.synchronize()
    x = d.block_solve(F, rhs)
    torch.cuda.synchronize()
    c = _lib.counters_read(); _lib.counters_reset(False)
    sc = np.zeros(EX, dtype=np.int32)
    rt.cudaMemcpy(sc.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(cap["cnt"] + 4 * (cap["n"] - EX)), 4 * EX, 2)
    roles = sc[4 + 1024:4 + 2048]
    chain = np.nonzero(roles == 2)[0]
    print(f"it {it}: solve {c['union_ms'].get('solve', 0):.2f} ms; ptrs " + " ".join(f"{(v or 0) - 0x7f0000000000:x}" for v in cap["ptrs"]), flush=True)

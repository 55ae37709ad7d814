import sys, os, time, ctypes
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2002_05018_b200 import _lib
lib = _lib.load()
torch.cuda.init()
n = 1 << 20
srcs = [np.random.rand(n) + 1j * np.random.rand(n) for _ in range(3)]
pin = torch.empty(3 * n, dtype=torch.complex128, pin_memory=True)
flag = torch.zeros(1, dtype=torch.int32, pin_memory=True)
print("pin ptr", hex(pin.data_ptr()), "flag", hex(flag.data_ptr()), flush=True)
dev = torch.empty(3 * n, dtype=torch.complex128, device="cuda")
cs = torch.cuda.Stream()
csp = ctypes.c_void_p(cs.cuda_stream)
fptr = ctypes.c_void_p(flag.data_ptr())
H = _lib.hptr
for c in range(3):
    rc = lib.d3m_stream_wait_flag(fptr, c + 1, csp); print("wait rc", rc, flush=True)
    rc = lib.d3m_memcpy_batch(ctypes.c_void_p(dev.data_ptr()), ctypes.c_void_p(pin.data_ptr()), H(np.array([16*n*c])), H(np.array([16*n*c])), H(np.array([16*n])), 1, 1, csp)
    print("copy rc", rc, flush=True)
srcp = (ctypes.c_void_p * 3)(*[s.ctypes.data for s in srcs])
time.sleep(0.5)
print("flag before", flag.numpy()[0], "query", cs.query(), flush=True)
h = lib.d3m_host_stage_start(3, H(np.array([0, 1, 2, 3])), 3, srcp, H(np.array([0, 16*n, 32*n])), H(np.array([16*n]*3)), ctypes.c_void_p(pin.data_ptr()), fptr, 4)
print("handle", h, flush=True)
rc = lib.d3m_host_stage_join(ctypes.c_void_p(h)); print("join", rc, "flag", flag.numpy()[0], flush=True)
cs.synchronize()
got = dev.cpu().numpy()
pv = pin.numpy()
print("pin ok", [np.array_equal(pv[c*n:(c+1)*n], srcs[c]) for c in range(3)], "dev==pin", [np.array_equal(got[c*n:(c+1)*n], pv[c*n:(c+1)*n]) for c in range(3)], flush=True)
print("first", srcs[0][:2], pv[:2], got[:2], flush=True)
print("ok", all(np.array_equal(got[c*n:(c+1)*n], srcs[c]) for c in range(3)), flush=True)

"""ctypes binding of libd3m.so (the C ABI declared in include/d3m.h).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is present, every compute entry point raises ``D3MUnavailable``.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("D3M_LIB") or os.path.join(_HERE, "libd3m.so")   # D3M_LIB: A/B builds (dev aid)

P = ctypes.c_void_p
I32 = ctypes.c_int
I64 = ctypes.c_int64
F64 = ctypes.c_double

# name -> argtypes (restype int unless stated)
_SIGNATURES = {
    "d3m_abi_version": [],
    "d3m_bk_factor_batched": [I32, I32, P, I64, I32, F64, I32, P, P, P, P, P, P, P, P, P, P],
    "d3m_bk_cluster_max_n": [I32],
    "d3m_host_stage_join": [P],
    "d3m_stream_wait_flag": [P, I32, P],
    "d3m_plan_flow_items": [I32, P, P, P, P, P, I64, P, I64, P, P],
    "d3m_ldlt_solve_batched": [I32, I32, P, I64, P, I64, P, I64, P, I64, I32, I32, P, P],
    "d3m_zgemm_grouped": [I32, I32, P, P, P, P, I32, P, P],
    "d3m_zgemm_tma_panels": [P, I64, P, I64, I32, P, P, I32, P, P],
    "d3m_gemm_set_form": [I32],
    "d3m_block_residual": [I32, P, P, P, P, P, P, P, P, P],
    "d3m_nonzero_rows": [I32, I32, I32, P, P, P, P, P],
    "d3m_block_solve_dataflow": [I32, P, P, I32, I32, P, P, P, I32, P, P, P, P, P, P, P, P, I32, P],
    "d3m_schur_reduce_batched": [I32, I32, I32, I32, P, P, P, F64] + [P] * 14 + [P, I32, P, I32, P, P, P],
    "d3m_block_copy": [P, P, P, I32, I64, P],
    "d3m_gather_rows": [P, P, P, I64, I32, P],
    "d3m_ordered_average": [P, P, P, P, I64, P],
    "d3m_zero": [P, I64, P],
    "d3m_diag_sym_exact": [P, P, P, I32, P, P],
    "d3m_modulus_probe": [P, P, P, I64, P],
    "d3m_block_ldlt_exec": [I32, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, I64, P, P, P, P, P, P, P,
                            P, F64, I32, I32, I32, P, P, P, P, P, P],
    "d3m_diag_sym_flags": [P, P, P, P, I32, P, P],
    "d3m_memcpy_batch": [P, P, P, P, P, I32, I32, P],
    "d3m_block_solve_exec": [I32, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, I64, I32, P, P],
    "d3m_recover_batched": [I32, I32, I32, P, P, P, P, P, P, P, P, P, P, I64, P, P],
    "d3m_counters_read": [P, P, P],
    "d3m_bk_panel_batched": [I32, I32, P, I64, I32, F64, I32, P, P, P, P, P, P, P, P, P, P],
    "d3m_ldlt_solve_blocked_batched": [I32, I32, P, I64, P, I64, P, I64, P, I64, I32, I32, P, P, P],
    "d3m_sym_scan_batched": [I32, I32, P, I64, I32, P, P, P, P],
    "d3m_copy_triangle": [I32, P, I64, P, I64, I64, I32, I32, I32, P],
}
_SIZE_T = {"d3m_bk_panel_workspace": [I32, I32]}
_PTR = {"d3m_host_stage_start": [I32, P, I32, P, P, P, P, P, I32]}
_INT64 = {"d3m_timing_intervals": [P, I64],
          "d3m_plan_gemm_tasks": [I32, P, P, P, P, P, P, I64, P, P, P, P, P]}
_VOID = {"d3m_set_timing": [I32], "d3m_counters_reset": []}

# GemmTask / CopyTask records (csrc/d3m_gemm.h, csrc/d3m_misc.h)
GEMM_TASK = np.dtype([("a_off", "<i8"), ("b_off", "<i8"), ("c_off", "<i8"), ("m", "<i4"), ("n", "<i4"),
                      ("k", "<i4"), ("lda", "<i4"), ("ldb", "<i4"), ("ldc", "<i4"), ("flags", "<i4"),
                      ("tile_start", "<i4"), ("tiles_n", "<i4"), ("pad", "<i4")])
assert GEMM_TASK.itemsize == 64
COPY_TASK = np.dtype([("src_off", "<i8"), ("dst_off", "<i8"), ("rows", "<i4"), ("cols", "<i4"),
                      ("ld_src", "<i4"), ("ld_dst", "<i4"), ("transpose", "<i4"), ("mode", "<i4")])
assert COPY_TASK.itemsize == 40

GEMM_SUB, GEMM_STORE, GEMM_ADD, GEMM_SYM = 0, 1, 2, 4
GEMM_TRIGATHER = 32       # csrc/d3m_gemm.h kGemmTriGather
TRSM_TRI_MAX = 512        # d3m_capi.cu kTrsmTriMax
COPY_STORE, COPY_ADD, COPY_ZERO_ADD = 0, 1, 2
GEMM_BM = GEMM_BN = 64
PANEL_BK_MIN = 512        # d3m_capi.cu kPanelBkMin


class D3MUnavailable(RuntimeError):
    """The CUDA extension or a CUDA device is missing: there is no fallback."""


class D3MError(RuntimeError):
    """A libd3m call returned an error code."""


_lib = None


FLOW_EXTRA_COUNTERS = 2052  # include/d3m.h D3M_FLOW_EXTRA_COUNTERS
ABI_VERSION = 13         # include/d3m.h D3M_ABI_VERSION this binding is written for


def load():
    """Load libd3m.so (built by build_ext / __graft_entry__.build; there is no
    implicit rebuild).  A library of another ABI version is rejected: an old
    build would take the new argument lists silently."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise D3MUnavailable(
            f"{LIB_PATH} is missing; build it with `python -m paper_2002_05018_b200.build_ext` "
            "(the D3M path has no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    lib.d3m_abi_version.restype = ctypes.c_int
    lib.d3m_abi_version.argtypes = []
    if lib.d3m_abi_version() != ABI_VERSION:
        raise D3MUnavailable(f"{LIB_PATH} has ABI version {lib.d3m_abi_version()}, this binding needs "
                             f"{ABI_VERSION}; rebuild it with `python -m paper_2002_05018_b200.build_ext --force`")
    for name, args in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    lib.d3m_last_error.restype = ctypes.c_char_p
    lib.d3m_last_error.argtypes = []
    for name, args in _INT64.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int64
    for name, args in _SIZE_T.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_size_t
    for name, args in _PTR.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_void_p
    for name, args in _VOID.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = None
    _lib = lib
    return lib


def exported_symbols() -> list[str]:
    return list(_SIGNATURES) + list(_VOID) + list(_SIZE_T) + list(_INT64) + list(_PTR) + ["d3m_last_error"]


CLASSES = ("bk", "trsm", "gemm", "solve", "misc")


def counters_reset(timing: bool = False) -> None:
    lib = load()
    lib.d3m_counters_reset()
    lib.d3m_set_timing(1 if timing else 0)


def timing_intervals() -> np.ndarray:
    """(class, start_ms, end_ms) rows of the launches timed before the last
    counters_read() (classes as CLASSES)."""
    lib = load()
    n = int(lib.d3m_timing_intervals(None, 0))
    out = np.zeros((max(n, 1), 3), dtype=np.float64)
    lib.d3m_timing_intervals(out.ctypes.data, n)
    return out[:n]


def counters_read() -> dict:
    """{'launches': int, 'ms': {class: ms}, 'n': {class: count}}"""
    lib = load()
    nl = ctypes.c_int64(0)
    ms = (ctypes.c_double * 10)()
    n = (ctypes.c_int64 * 5)()
    lib.d3m_counters_read(ctypes.byref(nl), ms, n)
    return {"launches": int(nl.value), "ms": dict(zip(CLASSES, list(ms)[:5])),
            "union_ms": dict(zip(CLASSES, list(ms)[5:])), "n": dict(zip(CLASSES, list(n)))}


def call(name: str, *args):
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.d3m_last_error().decode(errors="replace")
        raise D3MError(f"{name} returned {rc}: {msg}")
    return rc


def gemm_form(form: int = 0) -> int:
    """Set the grouped GEMM's complex product form (3 = Gauss 3M, 4 = 4M; 0
    only queries) for later launches in this process; returns the previous."""
    return int(load().d3m_gemm_set_form(int(form)))


def ptr(t) -> ctypes.c_void_p:
    """Device (torch) or host (numpy) buffer address."""
    if t is None:
        return ctypes.c_void_p(0)
    if isinstance(t, np.ndarray):
        return t.ctypes.data_as(ctypes.c_void_p)      # keeps the array alive with the pointer
    return ctypes.c_void_p(t.data_ptr())


def hptr(a: np.ndarray) -> ctypes.c_void_p:
    """Host pointer of a C-contiguous array; the returned object holds a
    reference to the array, so a temporary (hptr(np.asarray(...))) stays
    alive until the call that receives the pointer has returned."""
    assert a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.c_void_p)

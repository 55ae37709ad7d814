"""Device plumbing: torch owns HBM buffers and streams, libd3m does the math.

``DeviceArray`` is the numpy-compatible handle the drop-in API returns for
device-resident results (K_D, g_d, lambda, ...): downstream stages consume the
device tensor directly, while ``np.asarray(x)`` / arithmetic with numpy arrays
materialise a host copy on demand, so callers written against the reference's
numpy return values keep working.
"""

from __future__ import annotations

import numpy as np

from . import _lib

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise _lib.D3MUnavailable("no CUDA device: the D3M sm_100a path has no CPU fallback")
    _lib.load()
    return t


def stream_ptr():
    t = torch()
    return _lib.ctypes.c_void_p(t.cuda.current_stream().cuda_stream)


def empty(shape, dtype="complex128"):
    t = require_cuda()
    return t.empty(shape, dtype=getattr(t, dtype), device="cuda")


def zeros(shape, dtype="complex128"):
    t = require_cuda()
    return t.zeros(shape, dtype=getattr(t, dtype), device="cuda")


def to_device(a, dtype=np.complex128):
    """Host array / DeviceArray / tensor -> contiguous CUDA tensor of `dtype`
    (the kernels read raw complex128 / int64 memory, so a tensor of another
    dtype is converted like np.asarray(a, dtype) would convert it; a tensor
    that already matches is passed through without a copy)."""
    t = require_cuda()
    if isinstance(a, DeviceArray):
        a = a.tensor
    if isinstance(a, t.Tensor):
        tdt = t.from_numpy(np.empty(0, dtype=dtype)).dtype
        if a.is_complex() and not tdt.is_complex:
            raise TypeError(f"cannot convert a {a.dtype} tensor to {np.dtype(dtype)}")
        return a.to(device="cuda", dtype=tdt).contiguous()
    arr = np.ascontiguousarray(np.asarray(a, dtype=dtype))
    return t.from_numpy(arr).to("cuda", non_blocking=False)


def upload_i64(a):
    t = require_cuda()
    return t.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.int64))).to("cuda")


def upload_bytes(a: np.ndarray):
    """Structured numpy array (task records) -> uint8 CUDA tensor."""
    t = require_cuda()
    raw = np.ascontiguousarray(a).view(np.uint8).reshape(-1)
    return t.from_numpy(raw.copy()).to("cuda")


def to_host(x) -> np.ndarray:
    t = torch()
    if isinstance(x, DeviceArray):
        return x.numpy()
    if isinstance(x, t.Tensor):
        return x.detach().cpu().numpy()
    return np.asarray(x)


class BatchHost:
    """Host copy of a batched device result shared by its per-item
    DeviceArrays (e.g. every K_D of one reduce batch): the first item read
    copies the whole batch with one D2H transfer into pinned memory, the
    others are views of it -- instead of one small pageable transfer per
    item (~3 GB/s at 2.4 MB)."""

    def __init__(self, tensor):
        self.tensor = tensor
        self._host = None

    def get(self) -> np.ndarray:
        if self._host is None:
            t = torch()
            h = t.empty(self.tensor.shape, dtype=self.tensor.dtype, pin_memory=True)
            h.copy_(self.tensor.detach(), non_blocking=True)
            t.cuda.current_stream().synchronize()
            self._host = h.numpy()
            self.tensor = None
        return self._host


class DeviceArray:
    """A CUDA tensor that behaves like the numpy array the reference returns.
    ``batch`` = (BatchHost, index): the tensor is item ``index`` of a batched
    result and host copies come from the batch's single transfer."""

    __array_priority__ = 1000

    def __init__(self, tensor, batch=None):
        self.tensor = tensor
        self._host = None
        self._batch = batch

    # numpy interop -------------------------------------------------------
    def numpy(self) -> np.ndarray:
        if self._host is None:
            if self._batch is not None:
                grp, idx = self._batch
                self._host = grp.get()[idx]
                self._batch = None
            else:
                self._host = self.tensor.detach().cpu().numpy()
        return self._host

    def __array__(self, dtype=None, copy=None):
        a = self.numpy()
        return a.astype(dtype) if dtype is not None else a

    @property
    def shape(self):
        return tuple(self.tensor.shape)

    @property
    def ndim(self):
        return self.tensor.dim()

    @property
    def size(self):
        return int(self.tensor.numel())

    @property
    def dtype(self):
        return np.dtype(np.complex128) if self.tensor.is_complex() else self.numpy().dtype

    def __len__(self):
        return self.shape[0]

    def __getitem__(self, idx):
        return self.numpy()[idx]

    def __getattr__(self, name):
        if name in ("tensor", "_host", "_batch"):
            raise AttributeError(name)
        return getattr(self.numpy(), name)

    def __repr__(self):
        return f"DeviceArray(shape={self.shape}, device={self.tensor.device})"

    # arithmetic delegates to the host copy (verification-side convenience)
    def _h(self, o):
        return o.numpy() if isinstance(o, DeviceArray) else o

    def __add__(self, o): return self.numpy() + self._h(o)
    def __radd__(self, o): return self._h(o) + self.numpy()
    def __sub__(self, o): return self.numpy() - self._h(o)
    def __rsub__(self, o): return self._h(o) - self.numpy()
    def __mul__(self, o): return self.numpy() * self._h(o)
    def __rmul__(self, o): return self._h(o) * self.numpy()
    def __truediv__(self, o): return self.numpy() / self._h(o)
    def __matmul__(self, o): return self.numpy() @ self._h(o)
    def __rmatmul__(self, o): return self._h(o) @ self.numpy()
    def __neg__(self): return -self.numpy()
    def __abs__(self): return np.abs(self.numpy())
    def __eq__(self, o): return self.numpy() == self._h(o)
    __hash__ = None

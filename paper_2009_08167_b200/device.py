"""Device plumbing: engine contexts bound to torch streams, zero-copy views.

PyTorch is used only to hold device vectors and to order work on streams;
every kernel on the hot path is the engine's own (libriga_b200.so).
"""
from __future__ import annotations

import ctypes
import threading

import numpy as np
import torch

from . import _lib

_tls = threading.local()


class Context:
    """An engine context (device, stream).  Wraps a torch stream so that
    torch allocations/copies and engine kernels are ordered on one stream."""

    def __init__(self, device: int | None = None, stream: torch.cuda.Stream | None = None, priority: int = 0):
        if not torch.cuda.is_available() or _lib.device_count() == 0:
            raise RuntimeError("no CUDA device visible: the B200 engine has no CPU fallback")
        if device is None:
            device = torch.cuda.current_device()
        self.device = int(device)
        self.stream = stream if stream is not None else torch.cuda.Stream(device=self.device, priority=priority)
        self.priority = priority
        h = ctypes.c_void_p()
        # torch's default stream has handle 0; the engine reads 0 as "make a
        # private stream", so pass cudaStreamLegacy (0x1) to stay ordered
        # with default-stream torch work
        raw = self.stream.cuda_stream or 1
        _lib.check(_lib.lib().riga_ctx_create(self.device, ctypes.c_void_p(raw), ctypes.byref(h)),
                   "ctx_create")
        self.handle = h

    def synchronize(self):
        _lib.check(_lib.lib().riga_ctx_synchronize(self.handle))

    def __enter__(self):
        self._prev = getattr(_tls, "ctx", None)
        _tls.ctx = self
        self._sc = torch.cuda.stream(self.stream)
        self._sc.__enter__()
        return self

    def __exit__(self, *exc):
        self._sc.__exit__(*exc)
        _tls.ctx = self._prev

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                _lib.lib().riga_ctx_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


_default: dict[int, Context] = {}
_dlock = threading.Lock()


def current() -> Context:
    """The context of the enclosing ``with Context(...)`` block, else a
    per-device default context on torch's current stream."""
    c = getattr(_tls, "ctx", None)
    if c is not None:
        return c
    dev = torch.cuda.current_device() if torch.cuda.is_available() else 0
    with _dlock:
        if dev not in _default:
            _default[dev] = Context(dev, torch.cuda.current_stream(dev))
        return _default[dev]


class Owned:
    """Owner of one engine handle, destroyed with it.  Zero-copy tensors of
    engine memory reference this (not the Python object that created it), so
    no reference cycle runs through a tensor -- torch holds its data owner
    in C++, out of reach of the cycle collector."""

    def __init__(self, handle, destroy: str):
        self.handle, self._destroy = handle, destroy

    def __del__(self):
        try:
            if self.handle:
                getattr(_lib.lib(), self._destroy)(self.handle)
                self.handle = None
        except Exception:
            pass


class _CAI:
    """__cuda_array_interface__ exporter for engine-owned memory."""

    def __init__(self, ptr: int, shape, strides=None, owner=None):
        self.__cuda_array_interface__ = {
            "shape": tuple(shape), "typestr": "<f8", "data": (int(ptr), False),
            "version": 3, "strides": strides, "stream": None}
        self._owner = owner


def wrap(ptr: int, shape, device: int, strides=None, owner=None) -> torch.Tensor:
    """Zero-copy float64 torch view of engine-owned device memory."""
    return torch.as_tensor(_CAI(ptr, shape, strides, owner), device=f"cuda:{device}")


def to_device(x, ctx: Context | None = None) -> torch.Tensor:
    ctx = ctx or current()
    if isinstance(x, torch.Tensor):
        if x.is_cuda and x.dtype == torch.float64 and x.is_contiguous():
            return x
        return x.to(device=f"cuda:{ctx.device}", dtype=torch.float64).contiguous()
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    with torch.cuda.stream(ctx.stream):
        return torch.from_numpy(a).to(f"cuda:{ctx.device}", non_blocking=False)


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu").numpy()


def mem_info(device: int = 0, reset_high: bool = False) -> dict:
    """Engine memory pool (stream-ordered allocations) of `device`, bytes."""
    out = np.zeros(4, dtype=np.int64)
    _lib.check(_lib.lib().riga_mem_info(int(device), int(bool(reset_high)), _lib.ptr(out)))
    return {"reserved": int(out[0]), "reserved_high": int(out[1]), "used": int(out[2]), "used_high": int(out[3])}

"""Device plumbing: torch provides HBM allocations and the CUDA stream; the
compute runs in libsketchpress_b200.so.  Fails loudly without a CUDA device
(there is no CPU path in this package)."""

from __future__ import annotations

import numpy as np

from .errors import SketchpressError

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


_cuda_ok = False


def require_cuda():
    """torch, once a CUDA device is known to exist (checked once: the NVML /
    environment probe of torch.cuda.is_available costs microseconds per call
    on the pipelines' host path)."""
    global _cuda_ok
    t = torch()
    if not _cuda_ok:
        if not t.cuda.is_available():
            raise SketchpressError(
                "paper_2105_01271_b200 runs on a CUDA (sm_100a) device; none is available "
                "(there is deliberately no CPU fallback)")
        _cuda_ok = True
    return t


def device():
    t = require_cuda()
    return t.device("cuda", t.cuda.current_device())


def stream_handle():
    t = require_cuda()
    return t.cuda.current_stream().cuda_stream


def ptr(x) -> int | None:
    """Raw device pointer of a torch tensor (None passes through as NULL)."""
    return None if x is None else x.data_ptr()


def empty(shape, dtype="f64"):
    t = require_cuda()
    td = t.float64 if dtype == "f64" else (t.float32 if dtype == "f32" else t.int64)
    try:
        return t.empty(shape, dtype=td, device="cuda")
    except t.OutOfMemoryError:
        # the library keeps its freed workspaces (csrc/workspace.cu, up to 64 GB of
        # free lists + the CUDA mempool behind them), which torch's allocator cannot
        # reclaim: hand them back and retry once
        from . import _lib
        _lib.release_workspaces()
        t.cuda.empty_cache()
        return t.empty(shape, dtype=td, device="cuda")


def zeros(shape, dtype="f64"):
    t = empty(shape, dtype)
    t.zero_()
    return t


def to_device(a, dtype=None):
    """Host array (or torch tensor) -> contiguous device tensor."""
    t = require_cuda()
    if isinstance(a, t.Tensor):
        x = a
    else:
        arr = np.ascontiguousarray(a if dtype is None else np.asarray(a, dtype=dtype))
        x = t.from_numpy(arr)
    if dtype is not None:
        x = x.to(dtype={np.float64: t.float64, np.float32: t.float32, np.int64: t.int64}[np.dtype(dtype).type])
    x = x.to(device(), non_blocking=False).contiguous()
    if x.dim() == 2 and x.shape[0] == 1 and x.stride(0) != x.shape[1]:
        x = x.clone(memory_format=t.contiguous_format)  # np.atleast_2d view: row stride 0
        if x.stride(0) != x.shape[1]:
            x = x.reshape(-1).clone().reshape(1, -1)
    return x


def to_host(x) -> np.ndarray:
    return x.detach().cpu().numpy()


# Page-locked result buffers.  A result array handed to the caller is a numpy
# view of a page-locked buffer leased from this pool; the lease object is the
# array's base, so the buffer goes back to the pool when the caller's last
# view of it is garbage-collected, and the next call's device -> host copy
# lands in memory that is already page-locked and already touched.  (A fresh
# pinned allocation per call costs ~0.18 s per GB on the B200 box's host --
# 300 ms of a cfg4 call for V alone, measured -- and torch's pinned caching
# allocator hands blocks back only after its stream events are processed, so
# the first several calls of a loop all allocate.)
_POOL_MIN = 1 << 20          # smaller results: torch's pinned allocator
_POOL_KEEP = 2               # free buffers kept per size class
_POOL_CAP = 8 << 30          # free bytes kept in total
_pool: dict = {}
_pool_bytes = 0
_dt_str = {"torch.float64": "<f8", "torch.float32": "<f4", "torch.int64": "<i8", "torch.int32": "<i4",
           "torch.uint8": "|u1"}


def _size_class(nbytes: int) -> int:
    step = max(1 << 20, 1 << (max(nbytes, 1).bit_length() - 4))   # <= 12.5 % slack
    return (nbytes + step - 1) // step * step


class _Lease:
    """Owner of one leased buffer; exposes it through __array_interface__."""

    __slots__ = ("buf", "cls", "__array_interface__", "__weakref__")

    def __init__(self, buf, cls, shape, typestr):
        self.buf, self.cls = buf, cls
        self.__array_interface__ = {"shape": tuple(int(d) for d in shape), "typestr": typestr,
                                    "data": (buf.data_ptr(), False), "version": 3}

    def __del__(self):
        global _pool_bytes
        try:
            free = _pool.setdefault(self.cls, [])
            if len(free) < _POOL_KEEP and _pool_bytes + self.cls <= _POOL_CAP:
                free.append(self.buf)
                _pool_bytes += self.cls
        except Exception:      # interpreter shutdown
            pass


def _lease(t, nbytes: int):
    global _pool_bytes
    cls = _size_class(nbytes)
    free = _pool.get(cls)
    if free:
        _pool_bytes -= cls
        return free.pop(), cls
    return t.empty(cls, dtype=t.uint8, pin_memory=True), cls


def to_host_many(*xs):
    """Device tensors -> numpy arrays through page-locked buffers (one
    synchronisation for all; pageable D2H runs at a fraction of the link)."""
    t = torch()
    outs = []
    for x in xs:
        x = x.detach()
        nbytes = x.numel() * x.element_size()
        typestr = _dt_str.get(str(x.dtype))
        if nbytes < _POOL_MIN or typestr is None:
            h = t.empty(x.shape, dtype=x.dtype, pin_memory=True)
            h.copy_(x, non_blocking=True)
            outs.append(h)
            continue
        buf, cls = _lease(t, nbytes)
        h = buf[:nbytes].view(x.dtype).view(x.shape)
        h.copy_(x, non_blocking=True)
        outs.append(_Lease(buf, cls, x.shape, typestr))
    t.cuda.current_stream().synchronize()
    return [np.asarray(h) if isinstance(h, _Lease) else h.numpy() for h in outs]


def is_device_tensor(x) -> bool:
    t = torch()
    return isinstance(x, t.Tensor) and x.is_cuda


def synchronize():
    require_cuda().cuda.synchronize()

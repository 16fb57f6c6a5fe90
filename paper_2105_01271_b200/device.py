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


def to_host_many(*xs):
    """Device tensors -> numpy arrays through pinned staging buffers (one
    synchronisation for all; pageable D2H runs at a fraction of the link)."""
    t = torch()
    outs = []
    for x in xs:
        h = t.empty(x.shape, dtype=x.dtype, pin_memory=True)
        h.copy_(x.detach(), non_blocking=True)
        outs.append(h)
    t.cuda.current_stream().synchronize()
    return [h.numpy() for h in outs]


def is_device_tensor(x) -> bool:
    t = torch()
    return isinstance(x, t.Tensor) and x.is_cuda


def synchronize():
    require_cuda().cuda.synchronize()

"""The two metrics the hot path's callers use (src/analysis.py:57-74).

``rel_frob_error`` / ``oracle_error`` take host arrays like the reference.
``rel_frob_error_device`` evaluates ||A - U S V^T||_F / ||A||_F on the GPU
without forming the m x n reconstruction (K8), for A resident in HBM.
The rest of the reference's analysis module (theorem bounds, epsilon sweeps)
is out of scope.
"""

from __future__ import annotations

import numpy as np

from . import _lib


def rel_frob_error(a, approx) -> float:
    a = np.asarray(a, dtype=np.float64)
    approx = np.asarray(approx, dtype=np.float64)
    den = np.linalg.norm(a)
    if den == 0:
        return float(np.linalg.norm(approx))
    return float(np.linalg.norm(a - approx) / den)


def oracle_error(a, k: int) -> float:
    """Eckart-Young optimum ||A - A_k||_F / ||A||_F (host LAPACK; analysis only)."""
    s = np.linalg.svd(np.asarray(a, dtype=np.float64), compute_uv=False)
    tot = np.sqrt(np.sum(s ** 2))
    return float(np.sqrt(np.sum(s[k:] ** 2)) / tot) if tot > 0 else 0.0


def rel_frob_error_device(a_dev, u, s, v) -> float:
    """Streamed K8 on the GPU; a_dev is a CUDA tensor (f64/f32), u/s/v CUDA or host."""
    from .device import ptr, stream_handle, to_device
    u = u if hasattr(u, "is_cuda") else to_device(np.asarray(u, dtype=np.float64))
    s = s if hasattr(s, "is_cuda") else to_device(np.asarray(s, dtype=np.float64))
    v = v if hasattr(v, "is_cuda") else to_device(np.asarray(v, dtype=np.float64))
    u, s, v = u.contiguous(), s.contiguous(), v.contiguous()
    out = np.zeros(2)
    tag = _lib.SP_F64 if a_dev.dtype.itemsize == 8 else _lib.SP_F32
    k = u.shape[1]
    _lib.call("sp_frob_residual", ptr(a_dev), tag, a_dev.shape[0], a_dev.shape[1], a_dev.stride(0),
              ptr(u), k, ptr(s), ptr(v), k, k, out.ctypes.data_as(__import__("ctypes").c_void_p),
              stream_handle())
    return float(np.sqrt(out[0] / out[1])) if out[1] > 0 else float(np.sqrt(out[0]))

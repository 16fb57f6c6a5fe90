"""Dense kernels of the path on the GPU (src/kernels.py).

thin_qr   -> Householder TSQR (K4) + the reference sign convention
thin_svd  -> TSQR + one-sided Jacobi on the core (K5) + sign convention
pivoted_qr-> greedy MGS column pivoting with the reference tie-break (K7)
pinv_apply-> thresholded reciprocals (K6)

Host (numpy) inputs return numpy outputs; CUDA tensors return CUDA tensors.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigError, NumericalError

RANK_TOL = 1e-12  # src/kernels.py:19


@dataclass
class ThinQR:
    q: object
    r: object


@dataclass
class ThinSVD:
    u: object
    s: object
    v: object

    def rank(self, threshold: float = RANK_TOL) -> int:
        s = np.asarray(self.s.detach().cpu().numpy() if hasattr(self.s, "detach") else self.s)
        if s.size == 0 or s[0] <= 0.0:
            return 0
        return int(np.count_nonzero(s > threshold * s[0]))


@dataclass
class PivotedQR:
    q: object
    r: object
    perm: object


def _in(m):
    """-> (device f64 contiguous tensor, was_host)."""
    from .device import is_device_tensor, to_device, torch
    if is_device_tensor(m):
        x = m if m.dtype == torch().float64 else m.double()
        if x.dim() != 2:
            raise ConfigError("expected a 2-D matrix")
        return x.contiguous(), False
    arr = np.asarray(m, dtype=np.float64)
    if arr.ndim != 2:
        raise ConfigError("expected a 2-D matrix")
    return to_device(arr), True


def _out(x, host):
    from .device import to_host
    return to_host(x) if host else x


def _host_finite(x, what):
    from .device import torch
    if not bool(torch().isfinite(x).all()):
        raise NumericalError(f"{what} contains non-finite entries")


def thin_qr(m) -> ThinQR:
    """Reduced QR with the sign convention (src/kernels.py:74-84)."""
    from .device import empty, ptr, stream_handle
    x, host = _in(m)
    rows, cols = x.shape
    _host_finite(x, "QR input")
    p = min(rows, cols)
    q = empty((rows, p))
    r = empty((p, cols))
    _lib.call("sp_thin_qr", rows, cols, ptr(x), cols, ptr(q), p, ptr(r), cols, stream_handle())
    return ThinQR(q=_out(q, host), r=_out(r, host))


def thin_svd(m) -> ThinSVD:
    """Thin SVD (U, S, V) with V column-orthonormal (src/kernels.py:87-94)."""
    from .device import empty, ptr, stream_handle
    x, host = _in(m)
    rows, cols = x.shape
    _host_finite(x, "SVD input")
    p = min(rows, cols)
    u = empty((rows, p))
    s = empty((p,))
    v = empty((cols, p))
    _lib.call("sp_thin_svd", rows, cols, ptr(x), cols, ptr(u), p, ptr(s), ptr(v), p, stream_handle())
    return ThinSVD(u=_out(u, host), s=_out(s, host), v=_out(v, host))


def pivoted_qr(m, k: int) -> PivotedQR:
    """Rank-k column-pivoted QR, greedy on the largest residual norm with
    exact ties to the lowest original index (src/kernels.py:97-142)."""
    from .device import empty, ptr, stream_handle, torch
    x, host = _in(m)
    rows, cols = x.shape
    _host_finite(x, "pivoted QR input")
    if not 1 <= k <= min(rows, cols):
        raise ConfigError(f"rank k={k} outside [1, {min(rows, cols)}]")
    mt = x.t().contiguous()  # candidate columns contiguous
    perm = empty((cols,), "i64")
    q = empty((rows, k))
    r = empty((k, cols))
    _lib.call("sp_pivoted_qr", rows, cols, ptr(mt), rows, k, ptr(perm), ptr(q), k, ptr(r), cols,
              stream_handle())
    p = _out(perm, host)
    return PivotedQR(q=_out(q, host), r=_out(r, host), perm=p.astype(np.intp) if host else p)


def pinv_apply(s, threshold: float = RANK_TOL):
    """Reciprocals of singular values with a hard relative cutoff (src/kernels.py:158-168)."""
    from .device import empty, is_device_tensor, ptr, stream_handle, to_device, to_host
    dev = is_device_tensor(s)
    host_s = to_host(s) if dev else np.asarray(s, dtype=np.float64)
    if host_s.size and (np.any(host_s < 0) or np.any(np.diff(host_s) > 0)):
        raise ConfigError("singular values must be nonnegative and non-increasing")
    if host_s.size == 0:
        return s.clone() if dev else np.zeros_like(host_s)
    x = s.double().contiguous() if dev else to_device(host_s)
    out = empty(x.shape)
    _lib.call("sp_pinv_apply", ptr(x), x.numel(), float(threshold), ptr(out), stream_handle())
    return out if dev else to_host(out)


def lambda_max(sym) -> float:
    """Largest (signed) eigenvalue of a symmetric matrix (src/kernels.py:171-181):
    the reference's validation, then the one-sided Jacobi SVD of the shifted
    SPD matrix on the device (analysis._lambda_max_sym)."""
    from .analysis import _lambda_max_sym
    from .device import to_device
    a = np.asarray(sym.detach().cpu().numpy() if hasattr(sym, "detach") else sym, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ConfigError("lambda_max needs a square matrix")
    scale = max(1.0, np.max(np.abs(a))) if a.size else 1.0
    if a.size and np.max(np.abs(a - a.T)) > 1e-10 * scale:
        raise ConfigError("matrix is not symmetric to tolerance")
    if a.shape[0] == 0:
        return 0.0
    return _lambda_max_sym(to_device(a))


def numerical_rank(m, threshold: float = RANK_TOL) -> int:
    """Count of singular values above threshold * largest (src/kernels.py:191-196)."""
    return thin_svd(m).rank(threshold)


def spectral_norm(m) -> float:
    """Largest singular value (src/kernels.py:184-188)."""
    x = np.asarray(m, dtype=np.float64) if not hasattr(m, "detach") else m
    if getattr(x, "size", 1) == 0 or (hasattr(x, "numel") and x.numel() == 0):
        return 0.0
    s = thin_svd(m).s
    return float(s[0])

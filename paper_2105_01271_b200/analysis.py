"""Metrics and single-pass diagnostics around the hot path (src/analysis.py).

``rel_frob_error`` / ``oracle_error`` take host arrays like the reference.
``rel_frob_error_device`` evaluates ||A - U S V^T||_F / ||A||_F on the GPU
without forming the m x n reconstruction (K8), for A resident in HBM.
``verify_stream`` is the CLI ``--verify`` pass (src/cli.py:125-139) as one
extra streamed K8 read; ``reconstruct_blocks`` the device analogue of
``decompress_blocks`` (src/archive.py:269-276) on the factor pair.
``streaming_epsilon_sweep`` is SPC-ID-ERR (src/analysis.py:141-180) on the
device.  The theorem-bound evaluators stay out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigError


def rel_frob_error(a, approx) -> float:
    a = np.asarray(a, dtype=np.float64)
    approx = np.asarray(approx, dtype=np.float64)
    den = np.linalg.norm(a)
    if den == 0:
        return float(np.linalg.norm(approx))
    return float(np.linalg.norm(a - approx) / den)


def oracle_error(a, k: int) -> float:
    """Frobenius error of the best rank-k approximation, the singular-value
    tail ||A - A_k||_F (src/analysis.py:68-74; host LAPACK, analysis only)."""
    a = np.asarray(a, dtype=np.float64)
    if not 0 <= k <= min(a.shape):
        raise ConfigError(f"rank k={k} outside [0, {min(a.shape)}]")
    s = np.linalg.svd(a, compute_uv=False)
    return float(np.sqrt(np.sum(s[k:] ** 2)))


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


TAU_GRID_POINTS = 33     # src/analysis.py:24
TAU_GRID_SPAN = 100.0    # src/analysis.py:25


@dataclass
class TauSweep:
    """Gap values over a scale grid, with the grid minimiser (src/analysis.py:37-54)."""

    taus: np.ndarray
    values: np.ndarray
    sample_stride: int = 1

    @property
    def min_index(self) -> int:
        return int(np.argmin(self.values))

    @property
    def min_tau(self) -> float:
        return float(self.taus[self.min_index])

    @property
    def min_value(self) -> float:
        return float(self.values[self.min_index])


def factor_pair(result):
    """Left (m x k) and right (k x n) factors of a decomposition
    (src/archive.py:244-251); device tensors."""
    from .device import is_device_tensor, to_device
    from .svd import LowRankSVD

    def dev(x):
        return x.double().contiguous() if is_device_tensor(x) else to_device(np.asarray(x, dtype=np.float64))

    if isinstance(result, LowRankSVD):
        s = dev(result.s)
        return dev(result.u), (s[:, None] * dev(result.v).t()).contiguous()
    right = dev(result.skeleton)
    if result.lifting is not None:
        lift = result.lifting
        if hasattr(lift, "_dev_rmatmul"):  # FactoredLifting: (skel @ left) @ right factor, on device
            right = lift._dev_rmatmul(right)
        else:
            right = _mm(right, dev(lift))
    return dev(result.p), right


def _mm(a, b):
    from .device import empty, ptr, stream_handle
    out = empty((a.shape[0], b.shape[1]))
    _lib.call("sp_gemm", 0, 0, a.shape[0], b.shape[1], a.shape[1], 1.0, ptr(a), a.shape[1], ptr(b), b.shape[1],
              0.0, ptr(out), b.shape[1], stream_handle())
    return out


def reconstruct_blocks(left, right, block_rows: int = 256):
    """Yield reconstructed row blocks left[rows] @ right on the device
    without materialising the m x n matrix (decompress_blocks,
    src/archive.py:269-276)."""
    m = left.shape[0]
    if right.shape[0] != left.shape[1]:
        raise ConfigError("factor shapes disagree")
    for row in range(0, m, block_rows):
        yield _mm(left[row:row + block_rows].contiguous(), right)


def verify_stream(stream, result, block_rows: int = 256) -> dict:
    """The CLI --verify pass (src/cli.py:125-139): one more pass over the
    stream, ||A - left right||_F / ||A||_F accumulated by K8 without forming
    the reconstruction.  Returns {"rel_frob", "extra_passes": 1}."""
    from .device import ptr, stream_handle, to_device
    from .snapshot_io import DeviceSnapshotStream
    left, right = factor_pair(result)
    k = left.shape[1]
    ones = to_device(np.ones(max(k, 1)))
    v = right.t().contiguous()  # n x k
    passes0 = stream.passes_completed
    if stream.at_end_of_pass or stream.cursor != 0:
        stream.rewind()
    err = ref = 0.0
    st = stream_handle()
    out = np.zeros(2)
    optr = out.ctypes.data_as(__import__("ctypes").c_void_p)
    if isinstance(stream, DeviceSnapshotStream):
        a = stream.take_pass()
        tag = _lib.SP_F64 if a.dtype.itemsize == 8 else _lib.SP_F32
        _lib.call("sp_frob_residual", ptr(a), tag, stream.m, stream.n, a.stride(0), ptr(left), k, ptr(ones),
                  ptr(v), k, k, optr, st)
        err, ref = out[0], out[1]
    else:
        row = 0
        for blk in stream.blocks(block_rows):
            b = to_device(np.ascontiguousarray(blk, dtype=np.float64))
            rows = b.shape[0]
            _lib.call("sp_frob_residual", ptr(b), _lib.SP_F64, rows, stream.n, stream.n,
                      ptr(left[row:row + rows]), k, ptr(ones), ptr(v), k, k, optr, st)
            err += out[0]
            ref += out[1]
            row += rows
    rel = float(np.sqrt(err / ref)) if ref > 0 else float("nan")
    return {"rel_frob": rel, "extra_passes": stream.passes_completed - passes0}


def _lambda_max_sym(g):
    """Largest signed eigenvalue of a symmetric device matrix (n <= 256): the
    Jacobi SVD of the shifted SPD matrix g + s I, s = ||g||_F, minus s
    (src/kernels.py:171-181 uses eigvalsh)."""
    from .device import empty, ptr, stream_handle, torch
    t = torch()
    n = g.shape[0]
    if n == 0:
        return 0.0
    sh = float(t.linalg.matrix_norm(g).item())
    if sh == 0.0:
        return 0.0
    m = (g + g.t()) * 0.5 + sh * t.eye(n, dtype=g.dtype, device=g.device)
    u, s = empty((n, n)), empty((n,))
    _lib.call("sp_jacobi_svd", n, ptr(m), n, ptr(u), n, ptr(s), None, n, stream_handle())
    return float(s[0].item()) - sh


def streaming_epsilon_sweep(stream, op, m_c: int, taus=None, block_rows: int = 256):
    """SPC-ID-ERR (src/analysis.py:141-180): every c-th row (c = m // m_c,
    1-based rows i with i % c == 0, trailing remainder dropped) is kept on the
    fine grid and sketched, in one pass; the Gram gap lambda_max(B_f B_f^T -
    tau B_c B_c^T), scaled by c, over a tau grid (33-point log grid centred on
    (||B_f|| / ||B_c||)^2 by default).  Rows are gathered on the device (K1
    for the coarse side), the Grams on the DMMA GEMM, lambda_max by Jacobi."""
    from .device import empty, ptr, stream_handle, to_device
    from .snapshot_io import DeviceSnapshotStream, stage_stream
    if not 1 <= m_c <= stream.m:
        raise ConfigError(f"sampled row count m_c={m_c} outside [1, {stream.m}]")
    stride = stream.m // m_c
    rows = np.arange(stride - 1, stream.m, stride, dtype=np.int64)
    if rows.size > 256:
        raise ConfigError(f"streaming_epsilon_sweep keeps {rows.size} rows; the device path supports <= 256")
    st = stream_handle()
    staged = stage_stream(stream, block_rows)
    a = staged.a
    n = stream.n
    bf = empty((rows.size, n))
    d_rows = to_device(rows)
    _lib.call("sp_gather_rows", ptr(a), staged.dtype_tag, a.stride(0), n, ptr(d_rows), rows.size, ptr(bf), n, st)
    bc = empty((rows.size, op.out_dim))
    if op.idx is not None and op.omega is None:
        idx, w, depth, _ = op.device_tables()
        _lib.call("sp_apply_stencil", ptr(bf), _lib.SP_F64, rows.size, n, n, ptr(idx), ptr(w), depth, op.n_c, 0,
                  ptr(bc), op.n_c, st)
    else:
        from .sketch import apply_sketch
        bc = apply_sketch(op, bf)
    gf, gc = empty((rows.size, rows.size)), empty((rows.size, rows.size))
    for g, b, w_ in ((gf, bf, n), (gc, bc, bc.shape[1])):
        _lib.call("sp_gemm", 0, 1, rows.size, rows.size, w_, 1.0, ptr(b), w_, ptr(b), w_, 0.0, ptr(g), rows.size, st)
    if taus is None:
        top_f = np.sqrt(max(_lambda_max_sym(gf), 0.0))
        top_c = np.sqrt(max(_lambda_max_sym(gc), 0.0))
        if top_f == 0.0 or top_c == 0.0:
            raise ConfigError("tau grid needs nonzero fine and coarse matrices")
        center = (top_f / top_c) ** 2
        taus = np.geomspace(center / TAU_GRID_SPAN, center * TAU_GRID_SPAN, TAU_GRID_POINTS)
    taus = np.asarray(taus, dtype=np.float64)
    if taus.size == 0 or np.any(taus <= 0) or np.any(np.diff(taus) <= 0):
        raise ConfigError("tau grid must be positive and strictly increasing")
    values = np.array([stride * _lambda_max_sym(gf - t * gc) for t in taus])
    return TauSweep(taus=taus, values=values, sample_stride=stride)

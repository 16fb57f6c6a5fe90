"""Single-pass sketch SVD on the GPU (src/svd.py).

``single_pass_svd`` keeps the reference signature and result type.  One pass
of the stream stages A into HBM with the sketch gathered block by block as it
lands (K1); the sketch-sized factorisation (randomized subspace iteration,
TSQR, Jacobi) yields the kept left basis; one read of A (K2) forms A^T U_r;
TSQR + Jacobi of the r x r core give the factors.  Exact-arithmetic
equivalent of the reference's R^{-T} / pinv recovery.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigError, RankDeficiencyWarning
from .sketch import SketchOperator
from .snapshot_io import SnapshotStream, stage_stream

DEFAULT_BLOCK_ROWS = 256  # src/svd.py:28


@dataclass
class LowRankSVD:
    """Rank-k factors U (m x k), S (k,), V (n x k) (src/svd.py:31-43)."""

    u: object
    s: object
    v: object
    k: int
    method: str
    v_orthonormal: bool = True
    kept_rank: int | None = None  # effective rank of the projector (diagnostic)

    def reconstruct(self):
        return (self.u * self.s) @ self.v.T


def _validate_rank(k: int, op: SketchOperator, stream: SnapshotStream) -> None:
    # src/svd.py:71-77
    if k < 1:
        raise ConfigError("target rank k must be >= 1")
    if k > op.out_dim:
        raise ConfigError(f"target rank k={k} exceeds sketch width n_c={op.out_dim}")
    if k > min(stream.m, op.out_dim):
        raise ConfigError(f"target rank k={k} exceeds min(m, n_c)")


def _sketch_on_ingest(op: SketchOperator, m: int, cols=None, want_s0: bool = True, d_cols=None):
    """Buffers + per-block callback that gathers s0 = A D (and C = A(:, cols))
    from each block right after it lands in HBM (the fused ingest of K1)."""
    from .device import empty, ptr, stream_handle, to_device
    s0 = None
    c = None
    if op.idx is not None and want_s0:
        idx, w, depth, _ = op.device_tables()
        s0 = empty((m, op.n_c))
    if cols is not None:
        if d_cols is None:
            d_cols = to_device(np.asarray(cols, dtype=np.int64))
        c = empty((m, d_cols.numel()))

    def on_block(a, row0, rows):
        tag = _lib.SP_F64 if a.dtype.itemsize == 8 else _lib.SP_F32
        lda = a.stride(0)
        base = a[row0:row0 + rows]
        if s0 is not None:
            _lib.call("sp_apply_stencil", ptr(base), tag, rows, op.n, lda, ptr(idx), ptr(w), depth,
                      op.n_c, 0, ptr(s0[row0:row0 + rows]), op.n_c, stream_handle())
        if c is not None:
            nc = c.shape[1]
            _lib.call("sp_apply_stencil", ptr(base), tag, rows, op.n, lda, ptr(d_cols), None, 1, nc,
                      1, ptr(c[row0:row0 + rows]), nc, stream_handle())

    return s0, c, on_block


def _projected_s0(op: SketchOperator, staged, s0_coarse):
    """out_dim sketch: stencil (gathered on ingest) then omega, or a dense
    Gaussian operator (K3 GEMM)."""
    from .device import empty, ptr, stream_handle, to_device
    a = staged.a
    m = a.shape[0]
    if op.idx is None:  # dense gaussian kind: s0 = A @ dense
        ad = a if a.dtype.itemsize == 8 else a.double()
        dn = op.dense_device()
        s0 = empty((m, op.n_c))
        _lib.call("sp_gemm", 0, 0, m, op.n_c, op.n, 1.0, ptr(ad), ad.stride(0), ptr(dn), op.n_c, 0.0,
                  ptr(s0), op.n_c, stream_handle())
        s0_coarse = s0
    if op.omega is None:
        return s0_coarse
    om = to_device(np.ascontiguousarray(op.omega, dtype=np.float64))
    out = empty((m, op.out_dim))
    _lib.call("sp_gemm", 0, 0, m, op.out_dim, op.n_c, 1.0, ptr(s0_coarse), op.n_c, ptr(om), op.out_dim,
              0.0, ptr(out), op.out_dim, stream_handle())
    return out


def _finish(u, s, v, k, method, info, host, warn_msg):
    from .device import to_host_many
    if info[_lib.INFO_WARN] & _lib.SP_WARN_RANK_DEFICIENT:
        warnings.warn(warn_msg, RankDeficiencyWarning, stacklevel=3)
    if host:
        u, s, v = to_host_many(u, s, v)
    return LowRankSVD(u=u, s=s, v=v, k=k, method=method, kept_rank=int(info[_lib.INFO_KEPT]))


def accumulate_sketch(stream: SnapshotStream, op: SketchOperator,
                      block_rows: int = DEFAULT_BLOCK_ROWS, with_gram: bool = False,
                      return_device: bool = False):
    """One pass: coarse = A D (m x l) and optionally the literal cross-Gramian
    H = A^T (A D) (n x l) on the DMMA tensor pipe (src/svd.py:46-68)."""
    from .device import empty, ptr, stream_handle, to_host
    if op.n != stream.n:
        raise ConfigError(f"sketch fine dimension {op.n} != stream width {stream.n}")
    s0c, _, on_block = _sketch_on_ingest(op, stream.m)
    staged = stage_stream(stream, block_rows, on_block)
    coarse = _projected_s0(op, staged, s0c)
    gram = None
    if with_gram:
        a = staged.a if staged.a.dtype.itemsize == 8 else staged.a.double()
        l = coarse.shape[1]
        gram = empty((stream.n, l))
        _lib.call("sp_gemm", 1, 0, stream.n, l, stream.m, 1.0, ptr(a), a.stride(0), ptr(coarse), l, 0.0,
                  ptr(gram), l, stream_handle())
    if return_device:
        return coarse, gram
    return to_host(coarse), (None if gram is None else to_host(gram))


def single_pass_svd(stream: SnapshotStream, op: SketchOperator, k: int,
                    block_rows: int = DEFAULT_BLOCK_ROWS, return_device: bool = False) -> LowRankSVD:
    """SPC-SVD (src/svd.py:168-189): one pass, rank-k factors."""
    from .device import empty, ptr, stream_handle
    _validate_rank(k, op, stream)
    if op.n != stream.n:
        raise ConfigError(f"sketch fine dimension {op.n} != stream width {stream.n}")
    s0c, _, on_block = _sketch_on_ingest(op, stream.m)
    staged = stage_stream(stream, block_rows, on_block)
    s0 = _projected_s0(op, staged, s0c)
    m, n = stream.m, stream.n
    u, s, v = empty((m, k)), empty((k,)), empty((n, k))
    info = _lib.new_info()
    a = staged.a
    _lib.call("sp_single_pass_svd", ptr(a), staged.dtype_tag, m, n, a.stride(0), None, None, 1,
              op.out_dim, None, 0, k, ptr(s0), ptr(u), ptr(s), ptr(v), _lib.info_ptr(info),
              stream_handle())
    return _finish(u, s, v, k, "single_pass", info, not return_device,
                   "coarse sketch is rank deficient; using regularized triangular solve")


def two_pass_svd(stream: SnapshotStream, op: SketchOperator, k: int,
                 block_rows: int = DEFAULT_BLOCK_ROWS):
    raise NotImplementedError("two_pass_svd is a SURVEY 8(f) 'next' item; not in this build")


def direct_svd(stream: SnapshotStream, op: SketchOperator, k: int, p=None,
               block_rows: int = DEFAULT_BLOCK_ROWS):
    raise NotImplementedError("direct_svd is a SURVEY 8(f) 'next' item; not in this build")

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
from .errors import ConfigError, NumericalError, RankDeficiencyWarning
from .sketch import SketchOperator
from .snapshot_io import DeviceSnapshotStream, SnapshotStream, stage_stream

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


def _finish(u, s, v, k, method, info, host, warn_msg, rerun=None):
    """Warn / convert like the reference.  Host results: the fused finish's
    deferred device flag is read after the copies (no extra sync) and, if set,
    the call is re-run with the Householder finish (`rerun`), which reports
    non-finite data as NumericalError like the reference."""
    from .device import to_host_many
    if info[_lib.INFO_WARN] & _lib.SP_WARN_RANK_DEFICIENT:
        warnings.warn(warn_msg, RankDeficiencyWarning, stacklevel=3)
    if host:
        u_h, s_h, v_h = to_host_many(u, s, v)
        # only a call that took the fused finish has a deferred flag of its
        # own (a stale flag of an earlier return_device call is never read)
        if info[_lib.INFO_FUSED] and _lib.deferred_status() and rerun is not None:
            with _lib.householder_finish():
                rerun()
            if not np.all(np.isfinite(s.cpu().numpy())):
                raise NumericalError("non-finite values in the snapshot data")
            u_h, s_h, v_h = to_host_many(u, s, v)
        u, s, v = u_h, s_h, v_h
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

    def run():
        _lib.call("sp_single_pass_svd", ptr(a), staged.dtype_tag, m, n, a.stride(0), None, None, 1,
                  op.out_dim, None, 0, k, ptr(s0), ptr(u), ptr(s), ptr(v), _lib.info_ptr(info),
                  stream_handle())
    run()
    return _finish(u, s, v, k, "single_pass", info, not return_device,
                   "coarse sketch is rank deficient; using regularized triangular solve", rerun=run)


# ------------------------------------------------------------ second pass ----

def second_pass_atz(stream: SnapshotStream, z, block_rows: int = DEFAULT_BLOCK_ROWS):
    """One more pass over the stream: Y = A^T Z (n x l) on the device -- the
    ``projected += basis[rows].T @ block`` loops of the two-pass variants
    (src/svd.py:108-112, 135-140; src/power.py:149-154) with the result kept
    transposed.  A device-resident stream is one K2 call (TMA skinny pass for
    l <= 16, DMMA otherwise); host streams accumulate block by block in stream
    order on the DMMA GEMM (fixed order: reproducible)."""
    from .device import empty, ptr, stream_handle, to_device
    m, n, l = stream.m, stream.n, z.shape[1]
    y = empty((n, l))
    st = stream_handle()
    if isinstance(stream, DeviceSnapshotStream):
        a = stream.take_pass()
        tag = _lib.SP_F64 if a.dtype.itemsize == 8 else _lib.SP_F32
        _lib.call("sp_skinny_atz", ptr(a), tag, m, n, a.stride(0), ptr(z), l, l, ptr(y), l, st)
        return y
    row = 0
    for blk in stream.blocks(block_rows):
        b = to_device(np.ascontiguousarray(blk, dtype=np.float64))
        rows = b.shape[0]
        _lib.call("sp_gemm", 1, 0, n, l, rows, 1.0, ptr(b), n, ptr(z[row:row + rows]), l,
                  0.0 if row == 0 else 1.0, ptr(y), l, st)
        row += rows
    return y


def second_pass_rows(stream: SnapshotStream, indices, block_rows: int = DEFAULT_BLOCK_ROWS):
    """One more pass collecting the fine rows A[indices] (k x n, f64, order of
    ``indices`` kept): _gather_rows of src/rowid.py:82-95."""
    from .device import empty, is_device_tensor, ptr, stream_handle, to_device, to_host
    idx_h = to_host(indices) if is_device_tensor(indices) else np.asarray(indices)
    idx_h = idx_h.astype(np.int64)
    k, n = idx_h.size, stream.n
    if isinstance(stream, DeviceSnapshotStream):
        a = stream.take_pass()
        tag = _lib.SP_F64 if a.dtype.itemsize == 8 else _lib.SP_F32
        out = empty((k, n))
        d_idx = indices if is_device_tensor(indices) else to_device(idx_h)
        _lib.call("sp_gather_rows", ptr(a), tag, a.stride(0), n, ptr(d_idx), k, ptr(out), n, stream_handle())
        return out
    out_h = np.empty((k, n))
    order = np.argsort(idx_h, kind="stable")
    row = pos = 0
    for blk in stream.blocks(block_rows):
        hi = row + blk.shape[0]
        while pos < order.size and idx_h[order[pos]] < hi:
            out_h[order[pos]] = blk[idx_h[order[pos]] - row]
            pos += 1
        row = hi
    return to_device(out_h)


def _svd_of_projected_t(basis, y, k, method, host, v_orthonormal=True):
    """Rank-k SVD of projected = Y^T (l x n) and U = basis @ u_k
    (src/svd.py:141-143, src/power.py:115-121)."""
    from .device import empty, ptr, stream_handle, to_host_many
    n, l = y.shape
    st = stream_handle()
    if l > n:  # narrow stream: the ordinary thin SVD of the (tall) projected matrix
        from .kernels import thin_svd
        fac = thin_svd(y.t().contiguous())
        uu, ss, vv = fac.u, fac.s, fac.v
    else:
        uu, ss, vv = empty((l, l)), empty((l,)), empty((n, l))
        _lib.call("sp_thin_svd_t", l, n, ptr(y), l, ptr(uu), l, ptr(ss), ptr(vv), l, st)
    if ss.shape[0] < k:
        raise NumericalError(f"projected matrix supplies only {ss.shape[0]} directions")
    uk = uu[:, :k].contiguous()
    u = empty((basis.shape[0], k))
    _lib.call("sp_gemm", 0, 0, basis.shape[0], k, basis.shape[1], 1.0, ptr(basis), basis.shape[1], ptr(uk), k,
              0.0, ptr(u), k, st)
    s = ss[:k].clone()
    v = vv[:, :k].contiguous()
    if host:
        u, s, v = to_host_many(u, s, v)
    return LowRankSVD(u=u, s=s, v=v, k=k, method=method, v_orthonormal=v_orthonormal)


def two_pass_svd(stream: SnapshotStream, op: SketchOperator, k: int,
                 block_rows: int = DEFAULT_BLOCK_ROWS, return_device: bool = False) -> LowRankSVD:
    """Range basis from the sketch, projection in a second pass
    (src/svd.py:116-143): QR of the coarse sketch (K4), Y = A^T Q (K2 /
    DMMA), SVD of the projected matrix without transposing it (K4 + K5)."""
    from .device import to_host
    from .kernels import RANK_TOL, thin_qr, thin_svd
    _validate_rank(k, op, stream)
    coarse, _ = accumulate_sketch(stream, op, block_rows, return_device=True)
    s_coarse = to_host(thin_svd(coarse).s)
    achieved = int(np.count_nonzero(s_coarse > RANK_TOL * s_coarse[0])) if s_coarse[0] > 0 else 0
    if achieved < k:
        raise NumericalError(f"coarse matrix numerical rank {achieved} is below target rank {k}")
    basis = thin_qr(coarse).q
    stream.rewind()
    y = second_pass_atz(stream, basis, block_rows)
    return _svd_of_projected_t(basis, y, k, "two_pass", not return_device)


def direct_svd(stream: SnapshotStream, op: SketchOperator, k: int, p=None,
               block_rows: int = DEFAULT_BLOCK_ROWS, return_device: bool = False) -> LowRankSVD:
    """SVD of the sketch, right factors by a pseudo-inverse second pass
    (src/svd.py:80-113): V = (A^T U_k) / s_k, not orthonormal."""
    from .device import ptr, stream_handle, to_host, to_host_many
    from .kernels import RANK_TOL, thin_svd
    _validate_rank(k, op, stream)
    if p is None:
        p = op.out_dim - k
    if k + p != op.out_dim:
        raise ConfigError(f"sketch width {op.out_dim} != k + p = {k + p}")
    coarse, _ = accumulate_sketch(stream, op, block_rows, return_device=True)
    fac = thin_svd(coarse)
    s_h = to_host(fac.s)
    if s_h[k - 1] <= RANK_TOL * s_h[0]:
        raise NumericalError(f"coarse matrix numerical rank {fac.rank()} is below target rank {k}")
    u_k = fac.u[:, :k].contiguous()
    s_k = fac.s[:k].clone()
    stream.rewind()
    v = second_pass_atz(stream, u_k, block_rows)
    _lib.call("sp_scale_columns", stream.n, k, ptr(v), k, ptr(s_k), 1, stream_handle())
    if not return_device:
        u_k, s_k, v = to_host_many(u_k, s_k, v)
    return LowRankSVD(u=u_k, s=s_k, v=v, k=k, method="direct", v_orthonormal=False)

"""Single-pass power iteration on a column-subsampled Gramian, on the GPU
(src/power.py).

``power_svd`` / ``power_id`` keep the reference signatures.  In single-pass
mode the stream is read once into HBM with s0 = A D and C = A(:, I) gathered
per block (K1).  The SVD path then needs only the kept left basis of
G = (C C^T)^q s0 -- computed from C itself when s0 and C share the column
set (every BASELINE configuration), because then sigma(G) = sigma(C)^(2q+1)
and U_G = U_C -- and one read of A for A^T U_r (K2).  The ID path runs the
pivoted QR (K7) on the enriched sketch and returns the lifting factored.

``power_basis`` / ``finalize_svd`` are provided with the literal algebra on
the device for callers that use them directly.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ConfigError, NumericalError, RankDeficiencyWarning
from .kernels import RANK_TOL, thin_qr, thin_svd, pinv_apply
from .rowid import FactoredLifting, RowIDFactors
from .sketch import SketchOperator, _rng
from .snapshot_io import DeviceSnapshotStream, SnapshotStream, stage_stream
from .svd import (DEFAULT_BLOCK_ROWS, LowRankSVD, _finish, _projected_s0, _sketch_on_ingest, _svd_of_projected_t,
                  second_pass_atz, second_pass_rows)

SINGLE_PASS = "single_pass"
TWO_PASS = "two_pass"


@dataclass
class PowerConfig:
    """Settings for the subsampled-Gramian power iteration (src/power.py:34-67)."""

    q: int = 1
    columns: np.ndarray | None = None
    stride: int = 10
    reorth: bool = False
    mode: str = SINGLE_PASS
    tau: float | None = None

    def __post_init__(self):
        if self.q < 0:
            raise ConfigError("power iteration count q must be >= 0")
        if self.mode not in (SINGLE_PASS, TWO_PASS):
            raise ConfigError(f"unknown finalize mode {self.mode!r}")
        if self.stride < 1:
            raise ConfigError("column stride must be >= 1")
        if self.tau is not None and self.tau <= 0:
            raise ConfigError("tau must be positive")
        if self.mode == SINGLE_PASS and self.reorth:
            raise ConfigError("re-orthonormalization invalidates the single-pass finalize shortcut")

    def column_set(self, n: int) -> np.ndarray:
        if self.columns is not None:
            return np.asarray(self.columns, dtype=np.intp)
        return np.arange(0, n, self.stride, dtype=np.intp)


@dataclass
class RangeBasis:
    """Power-enriched orthonormal basis plus the no-power baseline (src/power.py:70-78)."""

    q_b: object
    r_b: object
    q_np: object
    q_iters: int
    reorth_used: bool = field(default=False)


def _validate_columns(cols: np.ndarray, k: int, out_dim: int, n: int) -> None:
    # src/power.py:216-224
    if cols.size == 0 or cols.min() < 0 or cols.max() >= n:
        raise ConfigError("column index set out of range")
    if cols.size <= k:
        raise ConfigError(f"column set size {cols.size} must exceed target rank {k}")
    if cols.size < out_dim:
        raise ConfigError(f"column set size {cols.size} must cover the sketch width {out_dim}")


def _distinct(cols):
    if np.unique(cols).size != cols.size:
        raise ConfigError("column indices must be distinct")


def _column_set_on_device(op: SketchOperator, cols: np.ndarray):
    """Validated device copy of the column set I, cached on the operator by
    content (the reference re-validates I on every block, src/sketch.py:206-210;
    the result only depends on I).  The last set is checked first by a plain
    comparison (no hash of the bytes) -- the repeated-call fast path."""
    last = op._dev.get("cols:last")
    if last is not None and last[2].shape == cols.shape and np.array_equal(last[2], cols):
        return last[0], last[1]
    key = ("cols", cols.size, hash(cols.tobytes()))
    hit = op._dev.get(key)
    if hit is not None and np.array_equal(hit[2], cols):
        op._dev["cols:last"] = hit
        return hit[0], hit[1]
    _distinct(cols)
    from .device import to_device
    d_cols = to_device(cols.astype(np.int64))
    same = op.is_injection_of(cols)
    op._dev[key] = (d_cols, same, cols.copy())
    op._dev["cols:last"] = op._dev[key]
    return d_cols, same


def power_svd(stream: SnapshotStream, op: SketchOperator, k: int, cfg: PowerConfig,
              block_rows: int = DEFAULT_BLOCK_ROWS, return_device: bool = False) -> LowRankSVD:
    """SPC-SVD with C-PWR enrichment (src/power.py:227-249): single-pass mode
    as one device pipeline; two-pass mode as power_basis + a second A pass."""
    from .device import empty, ptr, stream_handle, to_device
    if k > op.out_dim:
        raise ConfigError(f"target rank k={k} exceeds sketch width {op.out_dim}")
    cols = cfg.column_set(stream.n)
    _validate_columns(cols, k, op.out_dim, stream.n)
    if cfg.mode != SINGLE_PASS:
        return _power_svd_two_pass(stream, op, k, cfg, cols, block_rows, return_device)
    if cfg.q < 1:
        raise ConfigError("single-pass power pipeline needs q >= 1")
    d_cols, same = _column_set_on_device(op, cols)  # validates distinctness once per set
    if op.n != stream.n:
        raise ConfigError(f"block width {stream.n} != fine dimension {op.n}")
    # s0 == C for the BASELINE grids: gather the column block once -- on
    # ingest for host streams; for a device-resident A the pipeline gathers it
    # itself, fused with the range finder's first product (srht_gather)
    if same and isinstance(stream, DeviceSnapshotStream):
        s0c, c, on_block = None, None, None
    else:
        s0c, c, on_block = _sketch_on_ingest(op, stream.m, cols, want_s0=not same, d_cols=d_cols)
    staged = stage_stream(stream, block_rows, on_block)
    m, n = stream.m, stream.n
    s0 = c if same else _projected_s0(op, staged, s0c)
    if k < 1 or k > min(m, op.out_dim):
        raise ConfigError(f"target rank k={k} outside the enriched basis width")
    hints = _lib.SP_HINT_COLS_VALIDATED | (_lib.SP_HINT_SAME_SET if same else _lib.SP_HINT_DIFFERENT_SET)
    if op.idx is not None:
        idx, w, depth, om = op.device_tables()
    else:
        idx, w, depth, om = None, None, 0, None
    u, s, v = empty((m, k)), empty((k,)), empty((n, k))
    info = _lib.new_info()
    a = staged.a

    def run():
        _lib.call("sp_power_svd", ptr(a), staged.dtype_tag, m, n, a.stride(0), ptr(idx), ptr(w), depth,
                  op.n_c, ptr(om), (op.out_dim if om is not None else 0), ptr(d_cols), cols.size, cfg.q, k,
                  ptr(s0), ptr(c), hints, ptr(u), ptr(s), ptr(v), _lib.info_ptr(info), stream_handle())
    run()
    return _finish(u, s, v, k, "power", info, not return_device,
                   "enriched sketch is rank deficient; using regularized solve", rerun=run)


def _power_svd_two_pass(stream, op, k, cfg, cols, block_rows, return_device):
    """power_basis on the first pass's accumulators, projection in a second
    pass (src/power.py:243-249 with finalize_svd TWO_PASS, :143-156)."""
    d_cols, same = _column_set_on_device(op, cols)
    if op.n != stream.n:
        raise ConfigError(f"block width {stream.n} != fine dimension {op.n}")
    s0c, c, on_block = _sketch_on_ingest(op, stream.m, cols, want_s0=not same, d_cols=d_cols)
    staged = stage_stream(stream, block_rows, on_block)
    s0 = c if same else _projected_s0(op, staged, s0c)
    del staged
    basis = power_basis(c, s0, cfg)
    res = finalize_svd(basis, k, TWO_PASS, stream=stream, block_rows=block_rows, _device=True)
    if return_device:
        return res
    from .device import to_host_many
    u, s, v = to_host_many(res.u, res.s, res.v)
    return LowRankSVD(u=u, s=s, v=v, k=k, method=res.method)


def power_id(stream: SnapshotStream, op: SketchOperator, k: int, cfg: PowerConfig,
             r: int | None = None, block_rows: int = DEFAULT_BLOCK_ROWS,
             project_ell: int | None = None, project_seed: int = 0,
             return_device: bool = False) -> RowIDFactors:
    """Row ID with selection on the power-enriched sketch (src/power.py:252-308),
    single-pass mode.  The lifting is returned factored (FactoredLifting)."""
    if op.omega is not None:
        raise ConfigError("pass a plain sketch; use project_ell for the ID projection")
    if cfg.reorth:
        raise ConfigError("re-orthonormalization is not supported in the ID pipeline")
    if k > op.n_c:
        raise ConfigError(f"target rank k={k} exceeds sketch width n_c={op.n_c}")
    cols = cfg.column_set(stream.n)
    _validate_columns(cols, k, op.n_c, stream.n)
    _distinct(cols)
    if cfg.mode != SINGLE_PASS:
        return _power_id_two_pass(stream, op, k, cfg, cols, block_rows, project_ell, project_seed,
                                  return_device)
    return _run_id(stream, op, k, cols, cfg.q, r, block_rows, project_ell, project_seed,
                   False, "power", return_device)


def _power_id_two_pass(stream, op, k, cfg, cols, block_rows, project_ell, project_seed, return_device):
    """Selection on the enriched sketch (C C^T)^q (A D), fine skeleton rows
    gathered in a second pass (src/power.py:274-308, method power_two_pass)."""
    from .device import to_device
    from .rowid import _two_pass_factors, row_id
    if op.idx is None:
        raise ConfigError("the ID pipeline needs a stencil (deterministic) sketch")
    s0c, c, on_block = _sketch_on_ingest(op, stream.m, cols if cfg.q > 0 else None)
    staged = stage_stream(stream, block_rows, on_block)
    del staged
    enriched = _enrich(c, s0c, cfg.q)
    id_input = enriched
    if project_ell is not None:
        if not 1 <= project_ell < op.n_c:
            raise ConfigError(f"need 1 <= project_ell < n_c, got {project_ell}")
        omega = to_device(_rng(project_seed).standard_normal((op.n_c, project_ell)))
        id_input = _mm(0, 0, enriched, omega)
    picked = row_id(id_input, k)
    stream.rewind()
    skeleton = second_pass_rows(stream, picked.indices, block_rows)
    return _two_pass_factors(picked, skeleton, "power_two_pass", return_device)


def _run_id(stream, op, k, cols, q, r, block_rows, project_ell, project_seed, on_basis, method,
            return_device):
    from .device import empty, ptr, stream_handle, to_device, to_host
    if op.idx is None:
        raise ConfigError("the ID pipeline needs a stencil (deterministic) sketch")
    if project_ell is not None and not on_basis:
        if not 1 <= project_ell < op.n_c:
            raise ConfigError(f"need 1 <= project_ell < n_c, got {project_ell}")
    s0c, c, on_block = _sketch_on_ingest(op, stream.m, cols if q > 0 else None)
    staged = stage_stream(stream, block_rows, on_block)
    m, n = stream.m, stream.n
    if not 1 <= k <= min(m, op.n_c if not on_basis else k):
        raise ConfigError(f"rank k={k} outside [1, {min(m, op.n_c)}]")
    idx, w, depth, _ = op.device_tables()
    proj = None
    if project_ell is not None and not on_basis:
        proj = to_device(_rng(project_seed).standard_normal((op.n_c, project_ell)))
    r_req = int(r) if r is not None else 0
    if r is not None and r < k:
        raise ConfigError(f"lifting rank r={r} below target rank k={k}")
    r_max = max(r_req, 2 * k, 1)
    p = empty((m, k))
    ind = empty((k,), "i64")
    skel = empty((k, op.n_c))
    left = empty((op.n_c, r_max))
    # U_r^T A (r x n) is materialised unless it would crowd A out of HBM
    # (cfg5: 200 x 16.8M doubles = 27 GB beside a 134 GB A); then the right
    # factor stays implicit as (U_r, A) for a device-resident A.
    from .device import torch as _torch
    free_b, _ = _torch().cuda.mem_get_info()
    lazy = isinstance(stream, DeviceSnapshotStream) and r_max * n * 8 > free_b // 3
    right = None if lazy else empty((r_max, n))
    ur = empty((m, r_max)) if lazy else None
    info = _lib.new_info()
    d_cols = to_device(np.asarray(cols, dtype=np.int64)) if cols is not None else None
    a = staged.a
    _lib.call("sp_power_id", ptr(a), staged.dtype_tag, m, n, a.stride(0), ptr(idx), ptr(w), depth,
              op.n_c, ptr(d_cols), (0 if cols is None else len(cols)), q, k, r_req, ptr(proj),
              (project_ell or 0), int(on_basis), ptr(s0c), ptr(c), ptr(p), ptr(ind), ptr(skel),
              ptr(left), ptr(right), ptr(ur), r_max, _lib.info_ptr(info), stream_handle())
    warn = int(info[_lib.INFO_WARN])
    r_used = int(info[_lib.INFO_LIFT_R])
    rank = int(info[_lib.INFO_RANK])
    if warn & _lib.SP_WARN_ID_PINV:
        warnings.warn("ID pivots are rank deficient; using pseudo-inverse solve", RankDeficiencyWarning,
                      stacklevel=3)
    if warn & _lib.SP_WARN_LIFT_CLAMPED:
        req = r_req if r_req else max(k, min(2 * k, rank))
        warnings.warn(f"lifting rank {req} clamped to sketch rank {rank}", RankDeficiencyWarning,
                      stacklevel=3)
    if lazy:
        lifting = FactoredLifting(left[:, :r_used], None, host=not return_device, ur=ur[:, :r_used], a=a)
    else:
        lifting = FactoredLifting(left[:, :r_used], right[:r_used], host=not return_device)
    # device diagnostic: the rank-r split fell in a flat stretch of the sketch
    # spectrum too wide for the exact SVD
    lifting.bulk_split = bool(warn & _lib.SP_WARN_BULK_SPLIT)
    if return_device:
        return RowIDFactors(p=p, indices=ind, skeleton=skel, lifting=lifting, r=r_used, method=method)
    from .device import to_host_many
    hp, hind, hskel = to_host_many(p, ind, skel)
    return RowIDFactors(p=hp, indices=hind.astype(np.intp), skeleton=hskel, lifting=lifting, r=r_used,
                        method=method)


# --------------------------------------------------- literal API helpers ----

def _dev(x):
    from .device import is_device_tensor, to_device
    return (x.double().contiguous(), False) if is_device_tensor(x) else (to_device(np.asarray(x, dtype=np.float64)), True)


def _mm(ta, tb, a, b):
    """op(a) @ op(b) on the DMMA GEMM."""
    from .device import empty, ptr, stream_handle
    M = a.shape[1] if ta else a.shape[0]
    K = a.shape[0] if ta else a.shape[1]
    N = b.shape[0] if tb else b.shape[1]
    out = empty((M, N))
    _lib.call("sp_gemm", int(ta), int(tb), M, N, K, 1.0, ptr(a), a.shape[1], ptr(b), b.shape[1], 0.0,
              ptr(out), N, stream_handle())
    return out


def _exact_mm(ta, a, b_hi, b_lo):
    """op(a) (b_hi + b_lo) nearly exactly rounded, as a double-double (sp_gemm_exact)."""
    from .device import empty, ptr, stream_handle
    M = a.shape[1] if ta else a.shape[0]
    K = a.shape[0] if ta else a.shape[1]
    N = b_hi.shape[1]
    hi, lo = empty((M, N)), empty((M, N))
    _lib.call("sp_gemm_exact", int(ta), M, N, K, ptr(a), a.shape[1], ptr(b_hi), ptr(b_lo), N, ptr(hi), ptr(lo),
              N, stream_handle())
    return hi, lo


def _enrich(c, e, q):
    """(C C^T)^q e in the reference's association C (C^T e) (src/power.py:282-285),
    each product nearly exactly rounded with the iterate carried in
    double-double (the greedy pivots downstream are decided by ulp-level
    residual differences; see csrc/exact_gemm.cu).  When C^T e would not fit
    (|I| > m: cfg5) W = C C^T in plain FP64, as the device pipeline does."""
    if c.shape[1] > c.shape[0]:
        w = _mm(0, 1, c, c)
        for _ in range(q):
            e = _mm(0, 0, w, e)
            _check_growth(e)
        return e
    lo = None
    for _ in range(q):
        t_hi, t_lo = _exact_mm(1, c, e, lo)
        e, lo = _exact_mm(0, c, t_hi, t_lo)
        _check_growth(e)
    return e


def _check_growth(g):
    from .device import torch
    if not bool(torch().isfinite(g).all()):
        raise NumericalError("power iterate overflowed; enable re-orthonormalization (reorth)")


def power_basis(c, s0, cfg: PowerConfig) -> RangeBasis:
    """(C C^T)^q s0 then QR (src/power.py:88-112), literal association, on the GPU."""
    from .device import to_host
    cd, host = _dev(c)
    g, _ = _dev(s0)
    if cd.shape[0] != g.shape[0]:
        raise ConfigError("column subset and sketch must share the row dimension")
    s0d = g
    for _ in range(cfg.q):
        g = _mm(1, 0, cd, g)
        _check_growth(g)
        if cfg.reorth:
            g = thin_qr(g).q
        g = _mm(0, 0, cd, g)
        _check_growth(g)
        if cfg.reorth:
            g = thin_qr(g).q
    enriched = thin_qr(g)
    baseline = thin_qr(s0d)
    cv = (lambda x: to_host(x)) if host else (lambda x: x)
    return RangeBasis(q_b=cv(enriched.q), r_b=cv(enriched.r), q_np=cv(baseline.q), q_iters=cfg.q,
                      reorth_used=cfg.reorth)


def finalize_svd(basis: RangeBasis, k: int, mode: str, stream: SnapshotStream | None = None,
                 hc=None, c=None, s0=None, block_rows: int = DEFAULT_BLOCK_ROWS,
                 _device: bool = False) -> LowRankSVD:
    """Turn the enriched basis into a rank-k SVD (src/power.py:124-181), literal
    algebra on the GPU."""
    from .device import to_host
    qb_shape = basis.q_b.shape
    if k < 1 or k > qb_shape[1]:
        raise ConfigError(f"target rank k={k} outside the enriched basis width")
    if mode == TWO_PASS:
        if stream is None:
            raise ConfigError("two-pass finalize needs the stream")
        if stream.at_end_of_pass:
            stream.rewind()
        elif stream.cursor != 0:
            raise ConfigError("stream must be fresh or at end of pass")
        qb, host = _dev(basis.q_b)
        y = second_pass_atz(stream, qb, block_rows)  # projected^T = A^T Q_b
        return _svd_of_projected_t(qb, y, k, "power", host and not _device)
    if mode != SINGLE_PASS:
        raise ConfigError(f"unknown finalize mode {mode!r}")
    if basis.reorth_used:
        raise ConfigError("single-pass finalize is invalid after intermediate re-orthonormalization")
    if basis.q_iters < 1:
        raise ConfigError("single-pass finalize needs q >= 1; use single_pass_svd for q = 0")
    if hc is None or c is None or s0 is None:
        raise ConfigError("single-pass finalize needs the hc, c, and s0 accumulators")
    cd, host = _dev(c)
    s0d, _ = _dev(s0)
    hcd, _ = _dev(hc)
    qb, _ = _dev(basis.q_b)
    rb, _ = _dev(basis.r_b)
    right = _mm(1, 0, cd, s0d)
    ctc = _mm(1, 0, cd, cd)
    for _ in range(basis.q_iters - 1):
        right = _mm(0, 0, ctc, right)
    cross = _mm(0, 0, hcd, right)
    rb_h = to_host(rb)
    diag = np.abs(np.diag(rb_h))
    square = rb_h.shape[0] == rb_h.shape[1]
    if square and diag.size and diag.max() > 0 and diag.min() > RANK_TOL * diag.max():
        # R^{-T} cross^T  via  (R^{-1})^T: solve R X = I then multiply
        projected = _mm(0, 1, _inv_upper(rb), cross)
    else:
        warnings.warn("enriched sketch is rank deficient; using regularized solve", RankDeficiencyWarning,
                      stacklevel=2)
        fac = thin_svd(rb)
        sp = pinv_apply(fac.s)
        from .device import torch
        r_pinv = _mm(0, 1, fac.v * sp[None, :], fac.u)
        projected = _mm(0, 0, cross, r_pinv).t().contiguous()
    return _svd_from_projected(qb, projected, k, "power", host)


def _inv_upper(r):
    """R^{-T} as a matrix: X = R^{-1} I (device triangular solve), returned transposed."""
    from .device import empty, ptr, stream_handle, to_device
    kk = r.shape[0]
    eye = to_device(np.eye(kk))
    x = empty((kk, kk))
    _lib.call("sp_trsm_upper", kk, ptr(r), r.shape[1], kk, ptr(eye), kk, ptr(x), kk, stream_handle())
    return x.t().contiguous()


def _svd_from_projected(qb, projected, k, method, host):
    from .device import to_host
    fac = thin_svd(projected)
    if fac.s.shape[0] < k:
        raise NumericalError(f"projected matrix supplies only {fac.s.shape[0]} directions")
    u = _mm(0, 0, qb, fac.u[:, :k].contiguous())
    s = fac.s[:k].clone()
    v = fac.v[:, :k].contiguous()
    if host:
        u, s, v = to_host(u), to_host(s), to_host(v)
    return LowRankSVD(u=u, s=s, v=v, k=k, method=method)

"""numpy restatement of the sketchpress single-pass hot path (TEST ORACLE).

Test infrastructure only -- see ``oracle/__init__.py``.  Every routine below
restates one reference routine (``src/`` = ``/root/reference/pkg/src/sketchpress/``)
with the same arithmetic order where it matters for bit-exactness (the
stencil gather, the block-serial accumulation, the greedy pivot rule) and the
same LAPACK entry points elsewhere, so that on one host and one BLAS thread
count it reproduces the reference's outputs.  Pinned by
``tests/test_oracle_pins.py`` against ``tests/golden/*.npz``.
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass

import numpy as np
from scipy.linalg import solve_triangular

TOL = 1e-12  # src/kernels.py:19 (RANK_TOL)
BLOCK = 256  # src/svd.py:28 (DEFAULT_BLOCK_ROWS)


class OracleConfigError(ValueError):
    """Mirrors src/errors.py:8 ConfigError."""


class OracleNumericalError(ArithmeticError):
    """Mirrors src/errors.py:24 NumericalError."""


class OracleRankWarning(RuntimeWarning):
    """Mirrors src/errors.py:28 RankDeficiencyWarning."""


# ----------------------------------------------------------------------------
# dense kernels (src/kernels.py)
# ----------------------------------------------------------------------------

def sign_normalise(basis, companions=()):
    """src/kernels.py:52-71 -- make each column's first significant entry >= 0.

    ``companions`` holds (array, "col"|"row") pairs flipped alongside.
    """
    mag = np.abs(basis)
    for j in range(basis.shape[1]):
        top = mag[:, j].max() if basis.shape[0] else 0.0
        if top == 0.0:
            continue
        hits = np.flatnonzero(mag[:, j] > 1e-12 * top)
        first = hits[0] if hits.size else int(np.argmax(mag[:, j]))
        if basis[first, j] >= 0.0:
            continue
        basis[:, j] *= -1.0
        for arr, how in companions:
            if how == "col":
                arr[:, j] *= -1.0
            else:
                arr[j, :] *= -1.0


def _finite_or_raise(x, label):
    # src/kernels.py:47-49
    if not np.all(np.isfinite(x)):
        raise OracleNumericalError(f"{label} contains non-finite entries")


def qr_reduced(x):
    """src/kernels.py:74-84 -> (q, r) with the sign convention."""
    x = np.asarray(x, dtype=np.float64)
    _finite_or_raise(x, "QR input")
    q, r = np.linalg.qr(x, mode="reduced")
    sign_normalise(q, [(r, "row")])
    return q, r


def svd_thin(x):
    """src/kernels.py:87-94 -> (u, s, v) with v column-orthonormal."""
    x = np.asarray(x, dtype=np.float64)
    _finite_or_raise(x, "SVD input")
    u, s, vt = np.linalg.svd(x, full_matrices=False)
    v = np.ascontiguousarray(vt.T)
    sign_normalise(u, [(v, "col")])
    return u, s, v


def kept_rank(s, tol=TOL):
    """src/kernels.py:34-37 (ThinSVD.rank)."""
    if s.size == 0 or s[0] <= 0.0:
        return 0
    return int(np.count_nonzero(s > tol * s[0]))


def reciprocal_cut(s, tol=TOL):
    """src/kernels.py:158-168 (pinv_apply)."""
    s = np.asarray(s, dtype=np.float64)
    if s.size and (np.any(s < 0) or np.any(np.diff(s) > 0)):
        raise OracleConfigError("singular values must be nonnegative and non-increasing")
    inv = np.zeros_like(s)
    if s.size == 0 or s[0] == 0.0:
        return inv
    live = s > tol * s[0]
    inv[live] = 1.0 / s[live]
    return inv


def _unit_filler(basis):
    """src/kernels.py:145-155 -- first e_i with a large orthogonal residual."""
    rows = basis.shape[0]
    for i in range(rows):
        e = np.zeros(rows)
        e[i] = 1.0
        e -= basis @ (basis.T @ e)
        nrm = np.linalg.norm(e)
        if nrm > 0.5:
            return e / nrm
    raise OracleNumericalError("cannot extend orthonormal basis")


def greedy_pivoted_qr(x, k):
    """src/kernels.py:97-142 -- rank-k MGS column-pivoted QR.

    Residual norms recomputed every step; exact ties go to the smallest
    original column index; one re-orthogonalisation folded into R.
    Returns (q, r, perm).
    """
    x = np.asarray(x, dtype=np.float64)
    _finite_or_raise(x, "pivoted QR input")
    rows, cols = x.shape
    if not 1 <= k <= min(rows, cols):
        raise OracleConfigError(f"rank k={k} outside [1, {min(rows, cols)}]")
    w = x.copy()
    perm = np.arange(cols)
    q = np.zeros((rows, k))
    r = np.zeros((k, cols))
    for t in range(k):
        nrm = np.linalg.norm(w[:, t:], axis=0)
        top = nrm.max()
        cand = t + np.flatnonzero(nrm == top)
        j = cand[np.argmin(perm[cand])]
        if j != t:
            w[:, [t, j]] = w[:, [j, t]]
            r[:, [t, j]] = r[:, [j, t]]
            perm[[t, j]] = perm[[j, t]]
        v = w[:, t].copy()
        if t > 0:
            fix = q[:, :t].T @ v
            r[:t, t] += fix
            v -= q[:, :t] @ fix
        piv = np.linalg.norm(v)
        if piv == 0.0:
            v = _unit_filler(q[:, :t])
        else:
            v /= piv
        q[:, t] = v
        r[t, t] = piv
        if t + 1 < cols:
            proj = v @ w[:, t + 1:]
            r[t, t + 1:] = proj
            w[:, t + 1:] -= np.outer(v, proj)
    sign_normalise(q, [(r, "row")])
    return q, r, perm


# ----------------------------------------------------------------------------
# sketch operators (src/sketch.py)
# ----------------------------------------------------------------------------

def stencil_tables(kind, n, n_c, d=1, weights=None):
    """src/sketch.py:98-117,156-168 -- padded (depth, n_c) idx / w tables."""
    s = math.ceil(n / n_c)
    cols = []
    for j in range(n_c):
        if kind == "injection":
            cols.append((np.array([min(j * s, n - 1)]), np.array([1.0])))
        elif kind == "neighbor":
            wts = np.asarray(weights if weights is not None else (0.25, 0.5, 0.25), float)
            c = min(j * s, n - 1)
            ix = c + np.arange(-d, d + 1)
            ok = (ix >= 0) & (ix < n)
            ww = wts[ok]
            cols.append((ix[ok], ww / ww.sum()))
        elif kind == "global":
            lo = j * s
            if lo >= n:
                cols.append((np.array([n - 1]), np.array([1.0])))
            else:
                hi = min(lo + s, n)
                cols.append((np.arange(lo, hi), np.full(hi - lo, 1.0 / (hi - lo))))
        else:
            raise OracleConfigError(f"no stencil for kind {kind!r}")
    depth = max(c[0].size for c in cols)
    idx = np.zeros((depth, n_c), dtype=np.intp)
    w = np.zeros((depth, n_c))
    for j, (ix, ww) in enumerate(cols):
        idx[: ix.size, j] = ix
        w[: ww.size, j] = ww
    return idx, w


def grid_coarse_indices(shape, stride):
    """Flattened C-order indices of the coarse grid {all coords = 0 mod stride}.

    The BASELINE 2-D/3-D coarse grid; the reference has no
    builder for it and takes it as an explicit ``idx`` table (src/sketch.py:120-134).
    """
    axes = [np.arange(0, g, stride) for g in shape]
    mesh = np.meshgrid(*axes, indexing="ij")
    flat = np.zeros(mesh[0].shape, dtype=np.int64)
    for ax, g in zip(mesh, shape):
        flat = flat * g + ax
    return flat.ravel()


def sketch_rows(block, idx, w, dense=None, omega=None):
    """src/sketch.py:171-184 -- (rows, n) -> (rows, out_dim).

    Deterministic kinds sum ``block[:, idx[t]] * w[t]`` into zeros in stencil
    order t = 0, 1, ... (the product rounded, then the sum rounded).
    """
    block = np.atleast_2d(np.asarray(block, dtype=np.float64))
    if dense is not None:
        out = block @ dense
    else:
        out = np.zeros((block.shape[0], idx.shape[1]))
        for t in range(idx.shape[0]):
            out += block[:, idx[t]] * w[t]
    if omega is not None:
        out = out @ omega
    return out


def take_columns(block, cols):
    """src/sketch.py:201-211 (gather_columns) with its validation."""
    block = np.atleast_2d(np.asarray(block))
    cols = np.asarray(cols, dtype=np.intp)
    if cols.size == 0:
        raise OracleConfigError("empty column index set")
    if cols.min() < 0 or cols.max() >= block.shape[1]:
        raise OracleConfigError(f"column index out of range [0, {block.shape[1]})")
    if np.unique(cols).size != cols.size:
        raise OracleConfigError("column indices must be distinct")
    return block[:, cols]


# ----------------------------------------------------------------------------
# the one pass (src/svd.py:46-68, src/power.py:184-213)
# ----------------------------------------------------------------------------

def _row_blocks(a, block_rows):
    for lo in range(0, a.shape[0], block_rows):
        yield lo, a[lo:lo + block_rows]


def one_pass_sketch(a, idx, w, block_rows=BLOCK, with_gram=False, omega=None):
    """src/svd.py:46-68 -- coarse = A D (m x l) and optionally H = A^T (A D)."""
    m, n = a.shape
    out_dim = idx.shape[1] if omega is None else omega.shape[1]
    coarse = np.empty((m, out_dim))
    gram = np.zeros((n, out_dim)) if with_gram else None
    for lo, blk in _row_blocks(a, block_rows):
        piece = sketch_rows(blk, idx, w, omega=omega)
        coarse[lo:lo + blk.shape[0]] = piece
        if with_gram:
            gram += blk.T @ piece
    return coarse, gram


def one_pass_power(a, idx, w, cols, block_rows=BLOCK, coarse_gram=False,
                   column_gram=True, omega=None):
    """src/power.py:184-213 -- s0, C = A(:, I), optional coarse+H, optional H_c."""
    m, n = a.shape
    out_dim = idx.shape[1] if omega is None else omega.shape[1]
    s0 = np.empty((m, out_dim))
    c = np.empty((m, cols.size))
    coarse = np.empty((m, idx.shape[1])) if coarse_gram else None
    gram = np.zeros((n, idx.shape[1])) if coarse_gram else None
    hc = np.zeros((n, cols.size)) if column_gram else None
    for lo, blk in _row_blocks(a, block_rows):
        hi = lo + blk.shape[0]
        piece = sketch_rows(blk, idx, w, omega=omega)
        s0[lo:hi] = piece
        sub = take_columns(blk, cols)
        c[lo:hi] = sub
        if coarse_gram:
            coarse[lo:hi] = piece
            gram += blk.T @ piece
        if column_gram:
            hc += blk.T @ sub
    return s0, c, coarse, gram, hc


def accumulate_block_slab(blk, idx, w, cols, lo, hi, hc_slab=None):
    """One stream block of src/power.py:198-212 (the loop body of
    _power_accumulate, with_column_gram=True) restricted to the rows
    [lo, hi) of hc: s0 and C rows of the block and this block's contribution
    blk[:, lo:hi]^T C_blk to hc[lo:hi].  The block's work on every other hc
    row slab is identical in kind and independent, so timing one (block,
    slab) pair times a known fraction of the reference's accumulate pass --
    the CPU-baseline sample of bench.py at configurations whose full hc
    (n x |I|, 137 GB at cfg4) cannot be held.  ``hc_slab`` is the running
    accumulator (allocated once per pass, as the reference's hc is)."""
    piece = sketch_rows(blk, idx, w)
    sub = take_columns(blk, cols)
    if hc_slab is None:
        hc_slab = np.zeros((hi - lo, sub.shape[1]))
    hc_slab += blk[:, lo:hi].T @ sub          # the reference's in-place accumulation (:211)
    return piece, sub, hc_slab


# ----------------------------------------------------------------------------
# single-pass SVD (src/svd.py:146-189)
# ----------------------------------------------------------------------------

def _truncated_pinv(r):
    """V diag(pinv(s)) U^T of a triangular factor (src/svd.py:163-164)."""
    uu, ss, vv = svd_thin(r)
    return vv @ (reciprocal_cut(ss)[:, None] * uu.T)


def _healthy(r):
    d = np.abs(np.diag(r))
    return (r.shape[0] == r.shape[1] and d.size > 0 and d.max() > 0
            and d.min() > TOL * d.max())


def projected_from_cross(r, cross):
    """src/svd.py:146-165 / src/power.py:171-180: R^{-T} X^T or the pinv branch.

    Returns (projected, used_pinv).
    """
    if _healthy(r):
        return solve_triangular(r.T, cross.T, lower=True), False
    warnings.warn("sketch is rank deficient; using regularized solve", OracleRankWarning)
    return (cross @ _truncated_pinv(r)).T, True


@dataclass
class OracleSVD:
    u: np.ndarray
    s: np.ndarray
    v: np.ndarray
    k: int
    method: str
    used_pinv: bool = False
    kept: int = 0  # effective rank of the projector (pinv cut count, or l)

    def reconstruct(self):
        return (self.u * self.s) @ self.v.T


def _check_rank(k, out_dim, m):
    # src/svd.py:71-77
    if k < 1:
        raise OracleConfigError("target rank k must be >= 1")
    if k > out_dim:
        raise OracleConfigError(f"target rank k={k} exceeds sketch width n_c={out_dim}")
    if k > min(m, out_dim):
        raise OracleConfigError(f"target rank k={k} exceeds min(m, n_c)")


def _kept_of(r, used_pinv):
    if not used_pinv:
        return r.shape[0]
    return kept_rank(np.linalg.svd(r, compute_uv=False))


def spc_svd(a, idx, w, k, block_rows=BLOCK, omega=None):
    """src/svd.py:168-189 (single_pass_svd)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    out_dim = idx.shape[1] if omega is None else omega.shape[1]
    _check_rank(k, out_dim, a.shape[0])
    coarse, gram = one_pass_sketch(a, idx, w, block_rows, True, omega)
    q, r = qr_reduced(coarse)
    projected, used = projected_from_cross(r, gram)
    u, s, v = svd_thin(projected)
    if s.size < k:
        raise OracleNumericalError(f"projected matrix supplies only {s.size} directions")
    return OracleSVD(q @ u[:, :k], s[:k].copy(), v[:, :k].copy(), k, "single_pass",
                     used, _kept_of(r, used))


# ----------------------------------------------------------------------------
# single-pass power iteration (src/power.py)
# ----------------------------------------------------------------------------

def _finite_iterate(g):
    # src/power.py:81-85
    if not np.all(np.isfinite(g)):
        raise OracleNumericalError("power iterate overflowed; enable re-orthonormalization (reorth)")


def enrich_basis(c, s0, q):
    """src/power.py:88-112 without reorth: QR of G = (C C^T)^q s0 -> (Q_b, R_b)."""
    g = np.asarray(s0, dtype=np.float64).copy()
    for _ in range(q):
        g = c.T @ g
        _finite_iterate(g)
        g = c @ g
        _finite_iterate(g)
    return qr_reduced(g)


def _check_cols(cols, k, out_dim, n):
    # src/power.py:216-224
    if cols.size == 0 or cols.min() < 0 or cols.max() >= n:
        raise OracleConfigError("column index set out of range")
    if cols.size <= k:
        raise OracleConfigError(f"column set size {cols.size} must exceed target rank {k}")
    if cols.size < out_dim:
        raise OracleConfigError(f"column set size {cols.size} must cover the sketch width {out_dim}")


def spc_power_svd(a, idx, w, cols, k, q=1, block_rows=BLOCK, omega=None):
    """src/power.py:227-249 + 124-181 (power_svd, single_pass finalize)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    cols = np.asarray(cols, dtype=np.intp)
    out_dim = idx.shape[1] if omega is None else omega.shape[1]
    if k > out_dim:
        raise OracleConfigError(f"target rank k={k} exceeds sketch width {out_dim}")
    _check_cols(cols, k, out_dim, a.shape[1])
    if q < 1:
        raise OracleConfigError("single-pass power pipeline needs q >= 1")
    s0, c, _, _, hc = one_pass_power(a, idx, w, cols, block_rows, False, True, omega)
    qb, rb = enrich_basis(c, s0, q)
    if k < 1 or k > qb.shape[1]:
        raise OracleConfigError(f"target rank k={k} outside the enriched basis width")
    right = c.T @ s0
    ctc = c.T @ c
    for _ in range(q - 1):
        right = ctc @ right
    cross = hc @ right
    projected, used = projected_from_cross(rb, cross)
    u, s, v = svd_thin(projected)
    if s.size < k:
        raise OracleNumericalError(f"projected matrix supplies only {s.size} directions")
    return OracleSVD(qb @ u[:, :k], s[:k].copy(), v[:, :k].copy(), k, "power",
                     used, _kept_of(rb, used))


# ----------------------------------------------------------------------------
# interpolative decomposition (src/rowid.py, src/power.py:252-308)
# ----------------------------------------------------------------------------

@dataclass
class OracleID:
    p: np.ndarray
    indices: np.ndarray
    skeleton: np.ndarray
    lifting: np.ndarray | None
    r: int | None
    method: str
    pivot_gaps: np.ndarray | None = None

    def reconstruct(self):
        out = self.p @ self.skeleton
        return out if self.lifting is None else out @ self.lifting


def pivot_gaps(x, k):
    """Gaps only (see greedy_pivots_and_gaps)."""
    return greedy_pivots_and_gaps(x, k)[1]


def greedy_pivots_and_gaps(x, k):
    """(pivots, gaps): the first k greedy pivots of src/kernels.py:114-140 and
    the winner/runner-up residual-norm gap at each step, relative to the
    largest INITIAL column norm.

    Test helper for the pivot parity gate (SURVEY.md 8(c) gate 2): replays
    src/kernels.py:114-140 and records (best - second) / max_j ||x_j|| per
    step.  Rounding perturbs every residual norm by ~1e-16 of the initial
    scale, so a pivot is reproducible by any correct FP64 implementation only
    while this gap is far above that (the gate uses 1e-11).
    """
    x = np.asarray(x, dtype=np.float64)
    w = x.copy()
    rows, cols = w.shape
    q = np.zeros((rows, k))
    perm = np.arange(cols)
    gaps = np.zeros(k)
    scale = np.linalg.norm(w, axis=0).max()
    scale = scale if scale > 0 else 1.0
    for t in range(k):
        nrm = np.linalg.norm(w[:, t:], axis=0)
        order = np.argsort(-nrm, kind="stable")
        best = nrm[order[0]]
        second = nrm[order[1]] if order.size > 1 else 0.0
        gaps[t] = (best - second) / scale
        cand = t + np.flatnonzero(nrm == best)
        j = cand[np.argmin(perm[cand])]
        if j != t:
            w[:, [t, j]] = w[:, [j, t]]
            perm[[t, j]] = perm[[j, t]]
        v = w[:, t].copy()
        if t:
            v -= q[:, :t] @ (q[:, :t].T @ v)
        nv = np.linalg.norm(v)
        v = v / nv if nv > 0 else _unit_filler(q[:, :t])
        q[:, t] = v
        if t + 1 < cols:
            w[:, t + 1:] -= np.outer(v, v @ w[:, t + 1:])
    return perm[:k].copy(), gaps


def interp_rows(x, k):
    """src/rowid.py:53-79 (row_id)."""
    x = np.asarray(x, dtype=np.float64)
    rows, cols = x.shape
    if not 1 <= k <= min(rows, cols):
        raise OracleConfigError(f"rank k={k} outside [1, {min(rows, cols)}]")
    _, r, perm = greedy_pivoted_qr(x.T, k)
    r1, r2 = r[:, :k], r[:, k:]
    d = np.abs(np.diag(r1))
    if d.min() > TOL * max(d.max(), np.finfo(float).tiny):
        coef = solve_triangular(r1, r2)
    else:
        warnings.warn("ID pivots are rank deficient; using pseudo-inverse solve", OracleRankWarning)
        uu, ss, vv = svd_thin(r1)
        coef = vv @ (reciprocal_cut(ss)[:, None] * (uu.T @ r2))
    p = np.zeros((rows, k))
    p[perm[:k]] = np.eye(k)
    if k < rows:
        p[perm[k:]] = coef.T
    sel = perm[:k].copy()
    return OracleID(p, sel, x[sel].copy(), None, None, "direct")


def lift_operator(u, s, v, gram, r, k=None):
    """src/rowid.py:115-139 (build_lifting) -> (lifting, r_used)."""
    if k is not None and r < k:
        raise OracleConfigError(f"lifting rank r={r} below target rank k={k}")
    if r < 1:
        raise OracleConfigError("lifting rank r must be >= 1")
    rank = kept_rank(s)
    if r > rank:
        warnings.warn(f"lifting rank {r} clamped to sketch rank {rank}", OracleRankWarning)
        r = rank
    left = v @ (reciprocal_cut(s)[:, None] * (u.T @ u[:, :r]))
    return left @ (left.T @ gram.T), r


def spc_power_id(a, idx, w, cols, k, q=1, r=None, block_rows=BLOCK,
                 project_ell=None, project_seed=0):
    """src/power.py:252-308 (power_id, single_pass mode)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    cols = np.asarray(cols, dtype=np.intp)
    n_c = idx.shape[1]
    if k > n_c:
        raise OracleConfigError(f"target rank k={k} exceeds sketch width n_c={n_c}")
    _check_cols(cols, k, n_c, a.shape[1])
    _, c, coarse, gram, _ = one_pass_power(a, idx, w, cols, block_rows, True, False)
    enriched = coarse.copy()
    for _ in range(q):
        enriched = c @ (c.T @ enriched)
        _finite_iterate(enriched)
    sel_in = enriched
    if project_ell is not None:
        if not 1 <= project_ell < n_c:
            raise OracleConfigError(f"need 1 <= project_ell < n_c, got {project_ell}")
        om = np.random.Generator(np.random.Philox(project_seed)).standard_normal((n_c, project_ell))
        sel_in = enriched @ om
    picked = interp_rows(sel_in, k)
    u, s, v = svd_thin(coarse)
    rank = kept_rank(s)
    if r is None:
        r = max(k, min(2 * k, rank))
    lifting, _ = lift_operator(u, s, v, gram, r, k=k)
    out = OracleID(picked.p, picked.indices, coarse[picked.indices].copy(), lifting,
                   min(r, rank), "power")
    out.pivot_gaps = pivot_gaps(sel_in.T, k)
    return out


def spc_id(a, idx, w, k, r=None, block_rows=BLOCK, id_target="coarse",
           project_ell=None, project_seed=0):
    """src/rowid.py:142-183 (single_pass_id)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    n_c = idx.shape[1]
    if id_target not in ("coarse", "basis"):
        raise OracleConfigError(f"unknown id_target {id_target!r}")
    if k > n_c:
        raise OracleConfigError(f"target rank k={k} exceeds sketch width n_c={n_c}")
    coarse, gram = one_pass_sketch(a, idx, w, block_rows, True)
    u, s, v = svd_thin(coarse)
    rank = kept_rank(s)
    if r is None:
        r = max(k, min(2 * k, rank))
    lifting, _ = lift_operator(u, s, v, gram, r, k=k)
    sel_in = coarse if id_target == "coarse" else u[:, :k]
    if project_ell is not None and id_target == "coarse":
        if not 1 <= project_ell < n_c:
            raise OracleConfigError(f"need 1 <= project_ell < n_c, got {project_ell}")
        om = np.random.Generator(np.random.Philox(project_seed)).standard_normal((n_c, project_ell))
        sel_in = sel_in @ om
    picked = interp_rows(sel_in, k)
    return OracleID(picked.p, picked.indices, coarse[picked.indices].copy(), lifting,
                    min(r, rank), "single_pass")


# ----------------------------------------------------------------------------
# two-pass variants
# ----------------------------------------------------------------------------

def second_pass_project(a, z, block_rows=BLOCK):
    """The `projected += basis[rows].T @ block` loop (src/svd.py:108-112,
    135-140; src/power.py:149-154): Z^T A accumulated block by block."""
    out = np.zeros((z.shape[1], a.shape[1]))
    for lo, blk in _row_blocks(a, block_rows):
        out += z[lo:lo + blk.shape[0]].T @ blk
    return out


def direct_svd(a, idx, w, k, p=None, block_rows=BLOCK):
    """src/svd.py:80-113: SVD of the sketch, V by a pseudo-inverse pass."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    n_c = idx.shape[1]
    _check_rank(k, n_c, a.shape[0])
    if p is None:
        p = n_c - k
    if k + p != n_c:
        raise OracleConfigError(f"sketch width {n_c} != k + p = {k + p}")
    coarse, _ = one_pass_sketch(a, idx, w, block_rows)
    u, s, _ = svd_thin(coarse)
    if s[k - 1] <= TOL * s[0]:
        raise OracleNumericalError(f"coarse matrix numerical rank {kept_rank(s)} is below target rank {k}")
    vt = second_pass_project(a, u[:, :k], block_rows) / s[:k, None]
    return OracleSVD(u[:, :k].copy(), s[:k].copy(), vt.T.copy(), k, "direct")


def _svd_of_projected(basis, projected, k, method):
    """src/svd.py:141-143 / src/power.py:115-121."""
    u, s, v = svd_thin(projected)
    if s.size < k:
        raise OracleNumericalError(f"projected matrix supplies only {s.size} directions")
    return OracleSVD(basis @ u[:, :k], s[:k].copy(), v[:, :k].copy(), k, method)


def two_pass_svd(a, idx, w, k, block_rows=BLOCK):
    """src/svd.py:116-143: QR basis of the sketch, projection in pass two."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    _check_rank(k, idx.shape[1], a.shape[0])
    coarse, _ = one_pass_sketch(a, idx, w, block_rows)
    s = np.linalg.svd(coarse, compute_uv=False)
    achieved = int(np.count_nonzero(s > TOL * s[0])) if s[0] > 0 else 0
    if achieved < k:
        raise OracleNumericalError(f"coarse matrix numerical rank {achieved} is below target rank {k}")
    basis, _ = qr_reduced(coarse)
    return _svd_of_projected(basis, second_pass_project(a, basis, block_rows), k, "two_pass")


def gather_fine_rows(a, indices):
    """src/rowid.py:82-95 (_gather_rows): the rows, order of `indices` kept."""
    return np.ascontiguousarray(a, dtype=np.float64)[np.asarray(indices)].copy()


def two_pass_id(a, idx, w, k, block_rows=BLOCK):
    """src/rowid.py:98-112: row ID of the sketch, fine skeleton in pass two."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    if k > idx.shape[1]:
        raise OracleConfigError(f"target rank k={k} exceeds sketch width n_c={idx.shape[1]}")
    coarse, _ = one_pass_sketch(a, idx, w, block_rows)
    picked = interp_rows(coarse, k)
    return OracleID(picked.p, picked.indices, gather_fine_rows(a, picked.indices), None, None, "two_pass")


def power_svd_two_pass(a, idx, w, cols, k, q=1, block_rows=BLOCK):
    """src/power.py:227-249 with finalize_svd TWO_PASS (:143-156)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    cols = np.asarray(cols, dtype=np.intp)
    out_dim = idx.shape[1]
    if k > out_dim:
        raise OracleConfigError(f"target rank k={k} exceeds sketch width {out_dim}")
    _check_cols(cols, k, out_dim, a.shape[1])
    s0, c, _, _, _ = one_pass_power(a, idx, w, cols, block_rows, False, False)
    qb, _ = enrich_basis(c, s0, q)
    if k < 1 or k > qb.shape[1]:
        raise OracleConfigError(f"target rank k={k} outside the enriched basis width")
    return _svd_of_projected(qb, second_pass_project(a, qb, block_rows), k, "power")


def power_id_two_pass(a, idx, w, cols, k, q=1, block_rows=BLOCK, project_ell=None, project_seed=0):
    """src/power.py:252-308, two-pass mode: fine skeleton rows, method power_two_pass."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    cols = np.asarray(cols, dtype=np.intp)
    n_c = idx.shape[1]
    if k > n_c:
        raise OracleConfigError(f"target rank k={k} exceeds sketch width n_c={n_c}")
    _check_cols(cols, k, n_c, a.shape[1])
    _, c, coarse, _, _ = one_pass_power(a, idx, w, cols, block_rows, True, False)
    enriched = coarse.copy()
    for _ in range(q):
        enriched = c @ (c.T @ enriched)
        _finite_iterate(enriched)
    sel_in = enriched
    if project_ell is not None:
        if not 1 <= project_ell < n_c:
            raise OracleConfigError(f"need 1 <= project_ell < n_c, got {project_ell}")
        om = np.random.Generator(np.random.Philox(project_seed)).standard_normal((n_c, project_ell))
        sel_in = enriched @ om
    picked = interp_rows(sel_in, k)
    out = OracleID(picked.p, picked.indices, gather_fine_rows(a, picked.indices), None, None, "power_two_pass")
    out.pivot_gaps = pivot_gaps(sel_in.T, k)
    return out


# ----------------------------------------------------------------------------
# SPC-ID-ERR: the streamed Gram-gap sweep (src/analysis.py:117-180)
# ----------------------------------------------------------------------------

def lambda_max_sym(sym):
    """src/kernels.py:171-181 (largest signed eigenvalue, symmetrised)."""
    sym = np.asarray(sym, dtype=np.float64)
    if sym.shape[0] == 0:
        return 0.0
    return float(np.linalg.eigvalsh((sym + sym.T) / 2.0)[-1])


def epsilon_sweep(a, idx, w, m_c, taus=None, block_rows=BLOCK, points=33, span=100.0):
    """src/analysis.py:141-180 (streaming_epsilon_sweep) with the default grid
    of :128-138 (centre (||B_f||_2 / ||B_c||_2)^2, 33 log points, span 100)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    m = a.shape[0]
    if not 1 <= m_c <= m:
        raise OracleConfigError(f"sampled row count m_c={m_c} outside [1, {m}]")
    stride = m // m_c
    keep_f, keep_c = [], []
    for lo, blk in _row_blocks(a, block_rows):
        first = ((lo // stride) + 1) * stride - 1   # 1-based row i kept when i % stride == 0
        local = np.arange(first - lo, blk.shape[0], stride)
        if local.size:
            sub = blk[local]
            keep_f.append(sub.copy())
            keep_c.append(sketch_rows(sub, idx, w))
    bf, bc = np.vstack(keep_f), np.vstack(keep_c)
    if taus is None:
        top_f = np.linalg.svd(bf, compute_uv=False)[0]
        top_c = np.linalg.svd(bc, compute_uv=False)[0]
        centre = (top_f / top_c) ** 2
        taus = np.geomspace(centre / span, centre * span, points)
    taus = np.asarray(taus, dtype=np.float64)
    gf, gc = bf @ bf.T, bc @ bc.T
    vals = np.array([stride * lambda_max_sym(gf - t * gc) for t in taus])
    return taus, vals, stride


# ----------------------------------------------------------------------------
# metrics used by the parity gates (src/analysis.py:57-74)
# ----------------------------------------------------------------------------

def rel_frob(a, approx):
    """src/analysis.py:57-65."""
    den = np.linalg.norm(a)
    return float(np.linalg.norm(a - approx) / den) if den > 0 else float(np.linalg.norm(approx))


def eckart_young(s_all, r):
    """Optimal relative Frobenius error of a rank-r approximation (src/analysis.py:68-74)."""
    tot = np.sqrt(np.sum(s_all ** 2))
    return float(np.sqrt(np.sum(s_all[r:] ** 2)) / tot) if tot > 0 else 0.0


# ----------------------------------------------------------------------------
# exact-arithmetic target of the same projector (test oracle for the GPU path)
# ----------------------------------------------------------------------------

def projector_target_svd(a, c, k, power=1):
    """Dense-LAPACK evaluation of what the single-pass methods compute in exact
    arithmetic: the rank-k SVD of P_r A, P_r the
    projector onto the top r left singular vectors of C (power = 2q+1 when
    s0 == C), r = #{(s_i/s_1)^power > 1e-12}.  Returns (u, s, v, r)."""
    a = np.asarray(a, dtype=np.float64)
    uc, sc, _ = np.linalg.svd(np.asarray(c, dtype=np.float64), full_matrices=False)
    r = int(np.count_nonzero((sc / sc[0]) ** power > TOL)) if sc[0] > 0 else 0
    z = uc[:, :r]
    y = a.T @ z
    qy, ry = np.linalg.qr(y)
    ut, st, vt = np.linalg.svd(ry.T)
    kk = min(k, r)
    return (z @ ut)[:, :kk], st[:kk], (qy @ vt.T)[:, :kk], r


def principal_angle(x, y):
    """Largest principal angle between span(x) and span(y) (orthonormal
    columns, same count), via sin(theta) = ||(I - y y^T) x||_2 -- accurate
    down to 1e-16, unlike arccos of the cosines."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if x.size == 0:
        return 0.0
    resid = x - y @ (y.T @ x)
    s = np.linalg.norm(resid, 2)
    return float(np.arcsin(min(s, 1.0)))


__all__ = [name for name in dir() if not name.startswith("_")]

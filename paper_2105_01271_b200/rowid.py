"""Row interpolative decomposition on the GPU (src/rowid.py).

``row_id`` runs the column-pivoted QR (K7) on the transpose plus the
triangular / pseudo-inverse coefficient solve on the device.  The single-pass
variants return the lifting operator FACTORED,
T = (V_r S_r^{-1}) (U_r^T A)  (src/rowid.py:115-139; PAPER eq. for the lift),
because the dense n_c x n lifting is 8.6 GB at cfg3 and 35 TB at cfg5.
``FactoredLifting`` behaves like the dense matrix for ``x @ T``, ``T @ x``,
``.shape`` and ``np.asarray`` (materialisation only for small cases).
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigError, RankDeficiencyWarning
from .kernels import RANK_TOL, ThinSVD

ID_ON_COARSE = "coarse"
ID_ON_BASIS = "basis"


class FactoredLifting:
    """Lazy n_c x n operator T = left @ right, left = V_r S_r^{-1} (n_c x r).

    ``right`` = U_r^T A (r x n) when it was materialised; otherwise it stays
    implicit as (ur = U_r (m x r), a = the device-resident A) and every product
    with T streams A through the device kernels.
    """

    __array_priority__ = 1000

    def __init__(self, left, right, host: bool = True, ur=None, a=None):
        if right is None and (ur is None or a is None):
            raise ValueError("FactoredLifting needs right, or ur and a")
        self.left = left
        self.right = right
        self.ur = ur
        self.a = a
        self.host = host
        self._cache = {}

    @property
    def shape(self):
        n = self.right.shape[1] if self.right is not None else self.a.shape[1]
        return (self.left.shape[0], n)

    @property
    def rank(self) -> int:
        return self.left.shape[1]

    def _h(self, name, x):
        if not hasattr(x, "detach"):
            return x
        if name not in self._cache:
            from .device import to_host_many
            self._cache[name] = to_host_many(x)[0]
        return self._cache[name]

    # ---- implicit right factor: products with A on the device
    def _mm(self, ta, tb, a, b, M, N, K):
        from .device import empty, ptr, stream_handle
        # left / right may be column slices of wider buffers: pass the row stride
        a = a if a.stride(1) == 1 else a.contiguous()
        b = b if b.stride(1) == 1 else b.contiguous()
        out = empty((M, N))
        _lib.call("sp_gemm", ta, tb, M, N, K, 1.0, ptr(a), a.stride(0), ptr(b), b.stride(0), 0.0, ptr(out), N,
                  stream_handle())
        return out

    def _times_a(self, wt):
        """w @ A for w = wt^T (rows x m), wt (m x rows): one read of A per call
        (FP32 A: the A^T Z pass, 16 columns per read)."""
        from .device import empty, ptr, stream_handle
        m, n = self.a.shape
        rows = wt.shape[1]
        if self.a.dtype.itemsize == 8:
            return self._mm(1, 0, rows, n, m, wt, self.a)
        y = empty((n, rows))
        _lib.call("sp_skinny_atz", ptr(self.a), _lib.SP_F32, m, n, self.a.stride(0), ptr(wt), rows, rows, ptr(y),
                  rows, stream_handle())
        return y.t().contiguous()

    def _dev_rmatmul(self, xd):
        w1 = self._mm(0, 0, xd, self.left, xd.shape[0], self.left.shape[1], xd.shape[1])   # x L
        if self.right is not None:
            return self._mm(0, 0, w1, self.right, w1.shape[0], self.right.shape[1], w1.shape[1])
        wt = self._mm(0, 1, self.ur, w1, self.ur.shape[0], w1.shape[0], self.ur.shape[1])  # U_r (x L)^T
        return self._times_a(wt)

    def __rmatmul__(self, x):
        """x @ T = (x @ left) @ right."""
        if self.right is not None and self.host:
            return (np.asarray(x) @ self._h("l", self.left)) @ self._h("r", self.right)
        from .device import is_device_tensor, to_device, to_host
        xd = x.double().contiguous() if is_device_tensor(x) else to_device(np.atleast_2d(np.asarray(x, np.float64)))
        out = self._dev_rmatmul(xd)
        if is_device_tensor(x):
            return out
        out = to_host(out)
        return out[0] if np.asarray(x).ndim == 1 else out

    def __matmul__(self, x):
        """T @ x = left @ (right @ x)."""
        if self.right is not None:
            if self.host:
                return self._h("l", self.left) @ (self._h("r", self.right) @ np.asarray(x))
            return self.left @ (self.right @ x)
        if self.a.dtype.itemsize != 8:
            raise NotImplementedError("T @ x with an implicit right factor needs FP64 A")
        from .device import is_device_tensor, to_device, to_host
        xd = x.double() if is_device_tensor(x) else to_device(np.asarray(x, np.float64))
        col = xd.dim() == 1
        xd = (xd.reshape(-1, 1) if col else xd).contiguous()
        ax = self._mm(0, 0, self.a, xd, self.a.shape[0], xd.shape[1], self.a.shape[1])      # A x
        z = self._mm(1, 0, self.ur, ax, self.ur.shape[1], ax.shape[1], self.ur.shape[0])     # U_r^T A x
        out = self._mm(0, 0, self.left, z, self.left.shape[0], z.shape[1], z.shape[0])
        out = out[:, 0] if col else out
        return out if is_device_tensor(x) else to_host(out)

    def __array__(self, dtype=None, copy=None):
        if self.right is not None:
            dense = self._h("l", self.left) @ self._h("r", self.right)
        else:
            from .device import to_device, to_host
            eye = to_device(np.eye(self.left.shape[0]))
            dense = to_host(self._dev_rmatmul(eye))
        return dense if dtype is None else dense.astype(dtype)

    def dense(self):
        return np.asarray(self)


@dataclass
class RowIDFactors:
    """Coefficients, selected rows, skeleton, optional lifting (src/rowid.py:30-50)."""

    p: object
    indices: object
    skeleton: object
    lifting: object = None
    r: int | None = None
    method: str = "direct"

    def reconstruct(self):
        approx = self.p @ self.skeleton
        if self.lifting is not None:
            approx = approx @ self.lifting
        return approx


def row_id(matrix, k: int) -> RowIDFactors:
    """Rank-k row ID via column-pivoted QR of the transpose (src/rowid.py:53-79)."""
    from .device import empty, is_device_tensor, ptr, stream_handle, to_device, to_host
    dev = is_device_tensor(matrix)
    x = matrix.double().contiguous() if dev else to_device(np.asarray(matrix, dtype=np.float64))
    if x.dim() != 2:
        raise ConfigError("expected a 2-D matrix")
    rows, cols = x.shape
    if not 1 <= k <= min(rows, cols):
        raise ConfigError(f"rank k={k} outside [1, {min(rows, cols)}]")
    p = empty((rows, k))
    ind = empty((k,), "i64")
    info = _lib.new_info()
    _lib.call("sp_row_id", rows, cols, ptr(x), cols, k, ptr(p), ptr(ind), _lib.info_ptr(info), stream_handle())
    if info[_lib.INFO_WARN] & _lib.SP_WARN_ID_PINV:
        warnings.warn("ID pivots are rank deficient; using pseudo-inverse solve", RankDeficiencyWarning,
                      stacklevel=2)
    if dev:
        return RowIDFactors(p=p, indices=ind, skeleton=x[ind].clone())
    indices = to_host(ind).astype(np.intp)
    return RowIDFactors(p=to_host(p), indices=indices, skeleton=np.asarray(matrix, dtype=np.float64)[indices].copy())


def build_lifting(coarse_svd: ThinSVD, gram, r: int, k: int | None = None):
    """V S+ U^T U_r U_r^T U S+ V^T H^T (src/rowid.py:115-139), dense, on the GPU."""
    from .device import empty, ptr, stream_handle, to_device, to_host
    from .kernels import pinv_apply
    if k is not None and r < k:
        raise ConfigError(f"lifting rank r={r} below target rank k={k}")
    if r < 1:
        raise ConfigError("lifting rank r must be >= 1")
    rank = coarse_svd.rank()
    if r > rank:
        warnings.warn(f"lifting rank {r} clamped to sketch rank {rank}", RankDeficiencyWarning, stacklevel=2)
        r = rank
    u = to_device(np.asarray(coarse_svd.u, dtype=np.float64))
    v = to_device(np.asarray(coarse_svd.v, dtype=np.float64))
    s = np.asarray(coarse_svd.s, dtype=np.float64)
    sp = to_device(pinv_apply(s))
    g = to_device(np.asarray(gram, dtype=np.float64))
    n_c, p = v.shape
    st = stream_handle()

    def mm(ta, tb, a, b, M, N, K):
        out = empty((M, N))
        _lib.call("sp_gemm", ta, tb, M, N, K, 1.0, ptr(a), a.shape[1], ptr(b), b.shape[1], 0.0, ptr(out), N, st)
        return out

    utu = mm(1, 0, u, u[:, :r].contiguous(), p, r, u.shape[0])       # U^T U_r
    left = mm(0, 0, v, (sp[:, None] * utu).contiguous(), n_c, r, p)  # V S+ (U^T U_r)
    tmp = mm(1, 1, left, g, r, g.shape[0], n_c)                       # left^T H^T
    return to_host(mm(0, 0, left, tmp, n_c, g.shape[0], r))


def single_pass_id(stream, op, k: int, r: int | None = None, block_rows: int = 256,
                   id_target: str = ID_ON_COARSE, project_ell: int | None = None,
                   project_seed: int = 0, return_device: bool = False) -> RowIDFactors:
    """SPC-ID (src/rowid.py:142-183): selection on the coarse sketch (or its
    leading left singular vectors), factored lifting, one pass."""
    from .power import _run_id
    if op.omega is not None:
        raise ConfigError("pass a plain sketch; use project_ell for the ID projection")
    if id_target not in (ID_ON_COARSE, ID_ON_BASIS):
        raise ConfigError(f"unknown id_target {id_target!r}")
    if k > op.n_c:
        raise ConfigError(f"target rank k={k} exceeds sketch width n_c={op.n_c}")
    out = _run_id(stream, op, k, None, 0, r, block_rows,
                  project_ell if id_target == ID_ON_COARSE else None, project_seed,
                  id_target == ID_ON_BASIS, "single_pass", return_device)
    return out


def two_pass_id(stream, op, k: int, block_rows: int = 256, return_device: bool = False) -> RowIDFactors:
    """Row selection on the sketch (pass one), fine skeleton gathered in pass
    two (src/rowid.py:98-112)."""
    from .svd import accumulate_sketch, second_pass_rows
    if k > op.out_dim:
        raise ConfigError(f"target rank k={k} exceeds sketch width n_c={op.out_dim}")
    coarse, _ = accumulate_sketch(stream, op, block_rows, return_device=True)
    picked = row_id(coarse, k)
    stream.rewind()
    skeleton = second_pass_rows(stream, picked.indices, block_rows)
    return _two_pass_factors(picked, skeleton, "two_pass", return_device)


def _two_pass_factors(picked, skeleton, method, return_device):
    if return_device:
        return RowIDFactors(p=picked.p, indices=picked.indices, skeleton=skeleton, method=method)
    from .device import to_host_many
    hp, hind, hskel = to_host_many(picked.p, picked.indices, skeleton)
    return RowIDFactors(p=hp, indices=hind.astype(np.intp), skeleton=hskel, method=method)

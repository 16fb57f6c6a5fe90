"""Column-sharded single-pass power SVD across the GPUs of one node
(SURVEY.md 8(e)).

A is split by contiguous column slabs (x-slabs of the C-order flattened grid:
rank i owns columns [c_b, c_e)); the coarse-grid points of a slab live on
that rank, so the gather is local.  Exchange steps (the only NVLink traffic):

1. all-gather of the column blocks C_i -> C (m x |I|, 65 MB at cfg2);
2. the sketch basis U_{C,r} is computed redundantly and bitwise identically
   on every rank (deterministic kernels, identical input);
3. the local A pass Y_i = A_i^T U_r (the HBM-bound kernel, no communication);
4. TSQR across ranks: local QR Y_i = Q_i R_i, all-gather of the r x r R_i,
   QR of the stack (redundant), Q_Y,i = Q_i Q_top,i;
5. the r x r core SVD (redundant); U and S replicated, V stays sharded;
6. the V completion to rank k: rank 0 (which holds the top k global rows)
   factors it and broadcasts the r x (k-r) K'; rank i appends -V_i K'.

This handles the s0 == A(:, I) case (the BASELINE coarse grids) of
``power_svd(..., PowerConfig(q, columns=I))`` in single-pass mode.
The arithmetic is pluggable (``ops``) so the exchange logic is tested on CPU
with gloo (tests/test_sharded_cpu.py); ``DeviceOps`` is the product path
(C-ABI kernels + torch.distributed / NCCL).
"""

from __future__ import annotations

import numpy as np

from . import _lib

RANK_TOL = 1e-12


class TorchComm:
    """torch.distributed collectives on the ops' tensors (NCCL or gloo)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1

    def allgather_cols(self, x, ops):
        """Concatenate each rank's (m x w_i) block along columns, rank order."""
        if self.world == 1:
            return x
        import torch
        widths = torch.tensor([x.shape[1]], dtype=torch.int64, device=ops.tensor_device)
        ws = [torch.zeros_like(widths) for _ in range(self.world)]
        self.dist.all_gather(ws, widths, group=self.group)
        ws = [int(w.item()) for w in ws]
        wmax = max(ws)
        pad = ops.pad_cols(x, wmax)
        parts = [ops.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(parts, pad, group=self.group)
        return ops.cat_cols([p[:, :w] for p, w in zip(parts, ws)])

    def allreduce_sum(self, x, ops):
        if self.world == 1:
            return x
        x = ops.contig(x)
        self.dist.all_reduce(x, group=self.group)
        return x

    def allgather_rows(self, x, ops):
        if self.world == 1:
            return x
        parts = [ops.empty_like(x) for _ in range(self.world)]
        self.dist.all_gather(parts, ops.contig(x), group=self.group)
        return ops.cat_rows(parts)

    def broadcast(self, x, root, ops):
        if self.world == 1:
            return x
        x = ops.contig(x)
        self.dist.broadcast(x, root, group=self.group)
        return x


SEED0 = 0x5EED5EED      # the range-finder seed of the device svd_top (csrc/pipeline.cu)
KEEP_TOL = 1e-12        # src/kernels.py:19


def _validate_cols(cols, k: int, n_total=None) -> np.ndarray:
    """The global column set I of the sharded drivers: the checks of
    src/power.py:216-224 (range, size) and src/sketch.py:207-210 (distinct),
    plus ascending order -- each rank gathers its own slab's columns in index
    order, so an unsorted I would permute the all-gathered C (and the ID's
    skeleton / lifting rows) relative to I."""
    from .errors import ConfigError
    cols = np.asarray(cols, dtype=np.int64).ravel()
    if cols.size == 0 or cols.min() < 0 or (n_total is not None and cols.max() >= n_total):
        raise ConfigError("column index set out of range")
    if cols.size <= k:
        raise ConfigError(f"column set size {cols.size} must exceed target rank {k}")
    d = np.diff(cols)
    if np.any(d == 0) or np.unique(cols).size != cols.size:
        raise ConfigError("column indices must be distinct")
    if np.any(d < 0):
        raise ConfigError("the sharded drivers need an ascending column set")
    return cols


def _count_kept(hs, power):
    if hs.size == 0 or not hs[0] > 0:
        return 0
    return int(np.count_nonzero((hs / hs[0]) ** power > KEEP_TOL))


def distributed_sketch_basis(c_i, row0: int, ncols: int, power: float, comm, ops):
    """Kept left basis U_{C,r} of the column-sharded sketch C = [C_1 .. C_P]
    without gathering C: the randomized block subspace iteration of the device
    svd_top (csrc/pipeline.cu) with the exchanges confined to m x b and b x b
    blocks.

      Y   = sum_i C_i Omega_i          (allreduce, m x b; Omega_i = rows
                                        row0.. of the global test block)
      Q   = TSQR(Y)                    (replicated, bit-identical)
      Z_i = C_i^T Q = P_i R_i          (local TSQR leaf)
      R   = QR([R_1; ...; R_P])        (allgather of b x b factors)
      R^T = U_s S V_s^T  (Jacobi)      U_C = Q U_s

    Same block size, growth and stopping rules as the single-GPU svd_top, so
    world size 1 reproduces it.  Returns (U m x r, sigma (host), r)."""
    m, nci = c_i.shape
    p = min(m, ncols)
    if p <= 64:  # exact path of svd_top: gather the (small) sketch
        c_all = comm.allgather_cols(c_i, ops)
        return ops.sketch_basis(c_all, power)
    cap = min(p, 256)
    b = min(cap, ((max(32, 1 + 16) + 7) // 8) * 8)
    while True:
        om = ops.fill_uniform(nci, b, SEED0 + b, row0)
        y = comm.allreduce_sum(ops.matmul(c_i, om), ops)
        qy, _ = ops.tsqr(y)
        prev, kept_prev, grow = None, -1, False
        for itn in range(24):
            z = ops.matmul_tn(c_i, qy)                                  # n_c_i x b
            zp = ops.pad_rows(z, b)                                     # TSQR needs rows >= b
            pz, rz = ops.tsqr(zp)
            if comm.world > 1:
                r_stack = comm.allgather_rows(rz, ops)
                q_top, r_all = ops.tsqr(r_stack)
            else:
                q_top, r_all = None, rz
            us, sg = ops.svd_small_t(r_all)                             # R^T = U_s S V_s^T
            hs = ops.to_numpy(sg)
            kept = _count_kept(hs, power)
            if kept + 8 > b and b < cap:
                grow = True
                break
            conv = itn == 0 and kept > 0 and b - 8 > kept and hs[b - 8] <= 1e-8 * hs[kept - 1]
            if (not conv and itn >= 1 and kept == kept_prev and kept > 0 and b - 8 > kept
                    and (hs[b - 8] / hs[kept - 1]) ** (2.0 * itn + 2.0) <= 1e-12):
                conv = True
            if not conv and itn >= 1 and kept == kept_prev:
                chk = min(b, kept + 1)
                conv = bool(np.all(np.abs(hs[:chk] - prev[:chk]) <= 1e-14 * hs[0] + 1e-12 * hs[:chk]))
            if conv:
                break
            prev, kept_prev = hs, kept
            # one more subspace iteration from the Ritz vectors, as svd_top:
            # Y = C (Z U_s) = sum_i C_i (Z_i U_s)  (Z_i local, U_s replicated)
            p_i = ops.matmul(z, us)
            y = comm.allreduce_sum(ops.matmul(c_i, p_i), ops)
            qy, _ = ops.tsqr(y)
        if grow:
            b = min(cap, 2 * b)
            continue
        r = kept
        u = ops.matmul(qy, ops.cols(us, 0, max(r, 1)))
        return ops.cols(u, 0, r), hs[:r], r


def sharded_power_svd(a_local, c_begin: int, cols, k: int, q: int, comm, ops, n_total=None):
    """Rank-local part of the column-sharded single-pass power SVD.

    a_local: this rank's columns [c_begin, c_begin + n_i) of A (m x n_i).
    cols: the global, ascending column set I.  Returns (U m x k, S k, V_i
    n_i x k, kept_rank, rank_deficient_warning) with U, S replicated.
    ``n_total`` (optional): the global column count, for the range check.
    """
    cols = _validate_cols(cols, k, n_total)
    m, n_i = a_local.shape
    sel = (cols >= c_begin) & (cols < c_begin + n_i)
    c_i = ops.gather(a_local, cols[sel] - c_begin)
    ncols = cols.size
    row0 = int(np.count_nonzero(cols < c_begin))  # this rank's first coarse column (global index)
    z, s_c, r = distributed_sketch_basis(c_i, row0, ncols, 2.0 * q + 1.0, comm, ops)
    r_use = max(r, 0)
    u = ops.zeros((m, k))
    v = ops.zeros((n_i, k))
    s = np.zeros(k)
    kk = min(r_use, k)
    if r_use > 0:
        y_i = ops.atz(a_local, z)                                   # n_i x r (the A pass)
        kappa = s_c[0] / s_c[r_use - 1] if s_c[r_use - 1] > 0 else np.inf
        # local QR leaf: CholeskyQR2 without a host sync when the kept spectrum
        # is narrow (breakdown is checked once, with the result's copy-back)
        flag = ops.new_flag() if kappa < 1e6 else None
        while True:
            q_i, r_i = ops.qr_async(y_i, flag) if flag is not None else ops.tsqr(y_i)
            if comm.world > 1:
                r_stack = comm.allgather_rows(r_i, ops)             # (P r) x r
                q_top, r_y = ops.tsqr(r_stack)
                q_y = ops.matmul(q_i, ops.rows(q_top, comm.rank * r_use, (comm.rank + 1) * r_use))
            else:
                q_y, r_y = q_i, r_i
            # SVD of R_y^T via that of R_y: R_y = A S B^T  =>  R_y^T = B S A^T
            a_, s_core, b_ = ops.svd_small(r_y)
            uf = ops.matmul(z, b_)                                  # U = Z u~,  u~ = B
            vf = ops.matmul(q_y, a_)                                # V = Q_Y v~, v~ = A
            u = ops.set_cols(u, ops.cols(uf, 0, kk), 0)
            v = ops.set_cols(v, ops.cols(vf, 0, kk), 0)
            if flag is None:
                break
            # a breakdown on ANY rank redoes the leaf with Householder on all ranks
            bad = comm.allreduce_sum(ops.flag_value(flag), ops)
            if not ops.to_numpy(bad).any():
                break
            flag = None
        s[:kk] = ops.to_numpy(s_core)[:kk]
    if kk < k:
        u = ops.complete(u, kk, k)
        if comm.rank == 0:
            v, kp = ops.complete_root(v, kk, k)
        else:
            kp = ops.zeros((kk, k - kk))
        kp = comm.broadcast(kp, 0, ops)
        if comm.rank != 0:
            v = ops.complete_other(v, kk, k, kp)
    warn = not (m >= ncols and r == ncols)
    return u, s, v, r, warn


class DeviceOps:
    """Product arithmetic: the C-ABI kernels on CUDA tensors."""

    def __init__(self):
        from .device import device, require_cuda
        self.t = require_cuda()
        self.tensor_device = device()

    # --- plumbing
    def _s(self):
        return self.t.cuda.current_stream().cuda_stream

    def zeros(self, shape):
        return self.t.zeros(shape, dtype=self.t.float64, device=self.tensor_device)

    def empty_like(self, x):
        return self.t.empty_like(x)

    def contig(self, x):
        return x.contiguous()

    def pad_cols(self, x, w):
        out = self.zeros((x.shape[0], w))
        out[:, :x.shape[1]] = x
        return out

    def cat_cols(self, parts):
        return self.t.cat(parts, dim=1).contiguous()

    def cat_rows(self, parts):
        return self.t.cat(parts, dim=0).contiguous()

    def rows(self, x, a, b):
        return x[a:b].contiguous()

    def cols(self, x, a, b):
        return x[:, a:b].contiguous()

    def set_cols(self, x, blk, c0):
        x[:, c0:c0 + blk.shape[1]] = blk
        return x

    def to_numpy(self, x):
        return x.cpu().numpy()

    # --- kernels
    def gather(self, a, idx_local):
        n_c = int(idx_local.size)
        out = self.t.empty((a.shape[0], n_c), dtype=self.t.float64, device=self.tensor_device)
        if n_c:
            d_idx = self.t.from_numpy(np.ascontiguousarray(idx_local, dtype=np.int64)).to(self.tensor_device)
            tag = _lib.SP_F64 if a.dtype.itemsize == 8 else _lib.SP_F32
            _lib.call("sp_apply_stencil", a.data_ptr(), tag, a.shape[0], a.shape[1], a.stride(0), d_idx.data_ptr(),
                      None, 1, n_c, 1, out.data_ptr(), n_c, self._s())
        return out

    def pad_rows(self, x, r):
        if x.shape[0] >= r:
            return x
        out = self.zeros((r, x.shape[1]))
        out[:x.shape[0]] = x
        return out

    def fill_uniform(self, rows, cols, seed, row0):
        out = self.t.empty((max(rows, 1), cols), dtype=self.t.float64, device=self.tensor_device)[:rows]
        if rows:
            _lib.call("sp_fill_uniform", rows, cols, out.data_ptr(), cols, int(seed), int(row0), self._s())
        return out

    def matmul_tn(self, a, b):
        """a^T b"""
        kdim, m = a.shape
        n = b.shape[1]
        out = self.t.empty((m, n), dtype=self.t.float64, device=self.tensor_device)
        if kdim == 0:
            return out.zero_()
        _lib.call("sp_gemm", 1, 0, m, n, kdim, 1.0, a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0), 0.0,
                  out.data_ptr(), n, self._s())
        return out

    def new_flag(self):
        return self.t.zeros((1,), dtype=self.t.int32, device=self.tensor_device)

    def flag_value(self, flag):
        return flag.double()

    def qr_async(self, x, flag):
        rows, c = x.shape
        qm = self.t.empty((rows, c), dtype=self.t.float64, device=self.tensor_device)
        rm = self.t.empty((c, c), dtype=self.t.float64, device=self.tensor_device)
        x = x.contiguous()
        _lib.call("sp_cholqr2_async", rows, c, x.data_ptr(), c, qm.data_ptr(), c, rm.data_ptr(), c, flag.data_ptr(),
                  self._s())
        return qm, rm

    def tsqr(self, x):
        rows, c = x.shape
        qm = self.t.empty((rows, c), dtype=self.t.float64, device=self.tensor_device)
        rm = self.t.empty((c, c), dtype=self.t.float64, device=self.tensor_device)
        x = x.contiguous()
        _lib.call("sp_tsqr", rows, c, x.data_ptr(), c, qm.data_ptr(), c, rm.data_ptr(), c, self._s())
        return qm, rm

    def svd_small_t(self, mtx):
        """U, S of mtx^T (U only: the left vectors of the transpose)."""
        n = mtx.shape[0]
        mt = mtx.t().contiguous()
        u = self.t.empty((n, n), dtype=self.t.float64, device=self.tensor_device)
        s = self.t.empty((n,), dtype=self.t.float64, device=self.tensor_device)
        _lib.call("sp_jacobi_svd", n, mt.data_ptr(), n, u.data_ptr(), n, s.data_ptr(), None, n, self._s())
        return u, s

    def sketch_basis(self, c, power):
        m, nc = c.shape
        rmax = min(m, nc, 256)
        u = self.t.empty((m, rmax), dtype=self.t.float64, device=self.tensor_device)
        s = self.t.empty((rmax,), dtype=self.t.float64, device=self.tensor_device)
        info = _lib.new_info()
        _lib.call("sp_sketch_basis", c.data_ptr(), m, nc, nc, float(power), rmax, u.data_ptr(), rmax, s.data_ptr(),
                  _lib.info_ptr(info), self._s())
        r = min(int(info[_lib.INFO_KEPT]), rmax)
        return u[:, :r].contiguous(), s[:r].cpu().numpy(), r

    def atz(self, a, z):
        n = a.shape[1]
        r = z.shape[1]
        y = self.t.empty((n, r), dtype=self.t.float64, device=self.tensor_device)
        tag = _lib.SP_F64 if a.dtype.itemsize == 8 else _lib.SP_F32
        _lib.call("sp_skinny_atz", a.data_ptr(), tag, a.shape[0], n, a.stride(0), z.data_ptr(), r, r, y.data_ptr(), r,
                  self._s())
        return y

    def qr(self, x, well_conditioned):
        rows, c = x.shape
        qm = self.t.empty((rows, c), dtype=self.t.float64, device=self.tensor_device)
        rm = self.t.empty((c, c), dtype=self.t.float64, device=self.tensor_device)
        _lib.call("sp_qr_tall", rows, c, x.data_ptr(), c, qm.data_ptr(), c, rm.data_ptr(), c, int(well_conditioned),
                  self._s())
        return qm, rm

    def matmul(self, a, b):
        m, kdim = a.shape
        n = b.shape[1]
        out = self.t.empty((m, n), dtype=self.t.float64, device=self.tensor_device)
        _lib.call("sp_gemm", 0, 0, m, n, kdim, 1.0, a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0), 0.0,
                  out.data_ptr(), n, self._s())
        return out

    def svd_small(self, mtx):
        n = mtx.shape[0]
        u = self.t.empty((n, n), dtype=self.t.float64, device=self.tensor_device)
        s = self.t.empty((n,), dtype=self.t.float64, device=self.tensor_device)
        v = self.t.empty((n, n), dtype=self.t.float64, device=self.tensor_device)
        _lib.call("sp_jacobi_svd", n, mtx.data_ptr(), n, u.data_ptr(), n, s.data_ptr(), v.data_ptr(), n, self._s())
        return u, s, v

    def complete(self, x, r, k):
        _lib.call("sp_householder_complete", x.shape[0], r, k, x.data_ptr(), x.stride(0), None, self._s())
        return x

    def complete_root(self, x, r, k):
        kp = self.t.empty((r, k - r), dtype=self.t.float64, device=self.tensor_device)
        _lib.call("sp_householder_complete", x.shape[0], r, k, x.data_ptr(), x.stride(0),
                  kp.data_ptr() if r > 0 else None, self._s())
        return x, kp

    def power_id_local(self, a_local, c_all, cols, k, q, r=None):
        """sp_power_id on this shard with the all-gathered C as both the
        coarse sketch and the column block (no gather, no index validation)."""
        import warnings

        from .device import empty, ptr, to_device, to_host_many
        from .errors import RankDeficiencyWarning
        m, n_i = a_local.shape
        ncols = int(c_all.shape[1])
        c_all = self.contig(c_all)
        d_cols = to_device(np.asarray(cols, dtype=np.int64))
        w = self.t.ones(ncols, dtype=self.t.float64, device=c_all.device)
        r_req = int(r) if r is not None else 0
        r_max = max(r_req, 2 * k, 1)
        p, ind, skel = empty((m, k)), empty((k,), "i64"), empty((k, ncols))
        left, right = empty((ncols, r_max)), empty((r_max, n_i))
        info = _lib.new_info()
        tag = _lib.SP_F64 if a_local.dtype == self.t.float64 else _lib.SP_F32
        _lib.call("sp_power_id", ptr(a_local), tag, m, n_i, a_local.stride(0), ptr(d_cols), ptr(w), 1, ncols,
                  ptr(d_cols), ncols, q, k, r_req, None, 0, 0, ptr(c_all), ptr(c_all), ptr(p), ptr(ind),
                  ptr(skel), ptr(left), ptr(right), None, r_max, _lib.info_ptr(info), self._s())
        warn = int(info[_lib.INFO_WARN])
        if warn & _lib.SP_WARN_ID_PINV:
            warnings.warn("ID pivots are rank deficient; using pseudo-inverse solve", RankDeficiencyWarning,
                          stacklevel=3)
        r_used = int(info[_lib.INFO_LIFT_R])
        hp, hind, hskel, hleft = to_host_many(p, ind, skel, left[:, :r_used].contiguous())
        return hp, hind.astype(np.intp), hskel, hleft, right[:r_used], r_used

    def complete_other(self, x, r, k, kp):
        if r > 0:
            _lib.call("sp_gemm", 0, 0, x.shape[0], k - r, r, -1.0, x.data_ptr(), x.stride(0), kp.data_ptr(), k - r,
                      0.0, x[:, r:].data_ptr(), x.stride(0), self._s())
        return x


def sharded_power_id(a_local, c_begin: int, cols, k: int, q: int, comm, ops, r=None, n_total=None):
    """Rank-local part of the column-sharded single-pass power ID (SURVEY.md
    8(e) item 5, the all-gather variant): the coarse column block C_i is
    gathered locally and all-gathered (m x |I|, 4.2 GB at cfg5 -- small beside
    the enrichment's two 2.1-TFLOP products that follow), then every rank runs
    the selection on the same bytes with the same deterministic kernels, so
    P, the pivots, the skeleton and the lifting's left factor V_r S_r^-1 come
    out bitwise identical on every rank; the lifting's right factor U_r^T A_i
    is this rank's column slab of U_r^T A (the lifting is column-sharded like
    A).  BASELINE case s0 == A(:, I) (injection at the column set).

    Returns (P m x k, indices k, skeleton k x |I|, left |I| x r, right_i
    r x n_i, r) -- host arrays for the replicated parts, device for right_i
    when ops is DeviceOps."""
    cols = _validate_cols(cols, k, n_total)
    m, n_i = a_local.shape
    sel = (cols >= c_begin) & (cols < c_begin + n_i)
    c_i = ops.gather(a_local, cols[sel] - c_begin)
    c_all = comm.allgather_cols(c_i, ops)                 # m x |I|, global column order
    return ops.power_id_local(a_local, c_all, cols, k, q, r)


def shard_columns(n: int, world: int, rank: int, align: int = 1) -> tuple[int, int]:
    """Contiguous column slab of a rank (rounded to ``align`` columns)."""
    units = n // align
    b = (units * rank // world) * align
    e = (units * (rank + 1) // world) * align if rank + 1 < world else n
    return b, e

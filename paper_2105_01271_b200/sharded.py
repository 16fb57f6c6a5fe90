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

    def allgather_cols(self, x, ops, widths=None):
        """Concatenate each rank's (m x w_i) block along columns, rank order.
        ``widths`` (every rank's w_i, known to the caller from the column
        layout) avoids the width exchange and its host synchronisation."""
        if self.world == 1:
            return x
        if widths is None:
            import torch
            wt = torch.tensor([x.shape[1]], dtype=torch.int64, device=ops.tensor_device)
            ws = [torch.zeros_like(wt) for _ in range(self.world)]
            self.dist.all_gather(ws, wt, group=self.group)
            widths = [int(w.item()) for w in ws]
        ws = list(widths)
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

    def allreduce_max(self, x, ops):
        if self.world == 1:
            return x
        x = ops.contig(x)
        self.dist.all_reduce(x, op=self.dist.ReduceOp.MAX, group=self.group)
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


def distributed_sketch_basis(c_i, row0: int, ncols: int, power: float, comm, ops, need: int = -1,
                             widths=None, want_v: bool = False):
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
    world size 1 reproduces it.  ``need`` >= 0 is svd_top's ID mode (only the
    leading ``need`` triplets and whether the rank reaches them).  Returns
    (U m x r, sigma (host), r) -- r the kept count, U's width min(r, block) --
    and with ``want_v`` also V_i (n_ci x width), this rank's rows of the right
    singular vectors, from the Rayleigh-Ritz factors P_i (accurate for every
    kept sigma; C_i^T U S^-1 would lose eps sigma_1 / sigma_i)."""
    m, nci = c_i.shape
    p = min(m, ncols)
    if p <= 64:  # exact path of svd_top: gather the (small) sketch
        c_all = comm.allgather_cols(c_i, ops, widths)
        if not want_v:
            return ops.sketch_basis(c_all, power)
        u, sv, v = ops.svd_full(c_all)
        hs = ops.to_numpy(sv)
        r = _count_kept(hs, power)
        return ops.cols(u, 0, r), hs[:r], r, ops.cols(ops.rows(v, row0, row0 + nci), 0, r)
    cap = min(p, 256)
    b = min(cap, ((max(32, 1 + 16) + 7) // 8) * 8)
    while True:
        om = ops.fill_uniform(nci, b, SEED0 + b, row0)
        y = comm.allreduce_sum(ops.matmul(c_i, om), ops)
        qy, _ = ops.tsqr(y)
        prev, kept_prev, grow = None, -1, False
        itn = -1
        while itn < 23:
            itn += 1
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
            if kept + 8 > b and (need < 0 or kept < need + 8):
                if b >= cap:
                    from .errors import ConfigError
                    raise ConfigError(f"sketch numerical rank {kept} exceeds the sharded range finder's "
                                      f"{cap}-column block")
                grow = True
                break
            if need >= 0:
                # ID mode (svd_top's rule): the leading t = min(kept, need)
                # triplets must be converged as a subspace, rate
                # rho = sigma_{b-7} / sigma_t; grow the block when more than 8
                # further steps would be needed; at the largest block a flat
                # stretch is accepted and flagged (no exact fallback across ranks)
                t = min(kept, need)
                conv = t == 0
                if not conv:
                    rho = hs[b - 8] / hs[t - 1]
                    conv = (itn == 0 and rho <= 1e-8) or (itn >= 1 and kept_prev >= t
                                                         and rho ** (2.0 * itn + 2.0) <= 1e-12)
                    if not conv:
                        more = (np.log(1e-12) / np.log(rho) - 2.0) / 2.0 - itn if rho < 1.0 else 1e9
                        if more > 8.0:
                            if b < cap and rho <= 0.95:   # a flat stretch does not resolve with a wider block
                                grow = True
                                break
                            conv = True   # bulk split: approximate beyond the resolvable part
            else:
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
            # blind steps (svd_top's rule): up to two before the step at which
            # the rate test can first pass, at most six in a row -- one allreduce
            # of m x b each, no R-factor all-gather, Jacobi core or host decision.
            # hs is replicated, so every rank takes the same number.
            tt = kept if need < 0 else min(kept, need)
            blind = 0
            if tt > 0 and (need >= 0 or b - 8 > kept):
                rho = hs[b - 8] / hs[tt - 1]
                if 0.0 < rho < 1.0:
                    pass_at = int(np.ceil((np.log(1e-12) / np.log(rho) - 2.0) / 2.0))
                    blind = min(max(pass_at, 1) - 2 - itn, 6, 21 - itn)
            for _ in range(max(blind, 0)):
                zb = ops.matmul_tn(c_i, qy)
                y = comm.allreduce_sum(ops.matmul(c_i, zb), ops)
                qy, _ = ops.tsqr(y)
                itn += 1
        if grow:
            b = min(cap, 2 * b)
            continue
        r = kept
        w = min(r, b)
        if not want_v:
            u = ops.matmul(qy, ops.cols(us, 0, max(w, 1)))
            return ops.cols(u, 0, w), hs[:w], r
        # R = A S B^T  ->  R^T = B S A^T: U_C = Q B, V_C,i = P_i Q_top,i A
        a_, _, b_ = ops.svd_small(r_all)
        u = ops.matmul(qy, ops.cols(b_, 0, max(w, 1)))
        pi = ops.rows(pz, 0, nci)
        if q_top is not None:
            pi = ops.matmul(pi, ops.rows(q_top, comm.rank * b, (comm.rank + 1) * b))
        v_i = ops.matmul(pi, ops.cols(a_, 0, max(w, 1)))
        return ops.cols(u, 0, w), hs[:w], r, ops.cols(v_i, 0, w)


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

    # --- the sharded ID (exact enrichment levels, distributed pivoted QR)
    def exponents(self, x, axis):
        rows, cols = x.shape
        e = self.t.empty((rows if axis == 1 else cols,), dtype=self.t.int32, device=self.tensor_device)
        _lib.call("sp_exponents", int(axis), rows, cols, x.data_ptr(), x.stride(0), e.data_ptr(), self._s())
        return e

    def exact_plan(self, K):
        import ctypes
        b, n = ctypes.c_int32(0), ctypes.c_int32(0)
        _lib.call("sp_exact_plan", int(K), ctypes.byref(b), ctypes.byref(n))
        return int(b.value), int(n.value)

    def transpose(self, x):
        return x.t().contiguous()

    def exact_levels(self, ta, a, ea, b, eb, bits, nsl):
        M = a.shape[1] if ta else a.shape[0]
        K = a.shape[0] if ta else a.shape[1]
        N = b.shape[1]
        lv = self.t.empty((nsl, M, N), dtype=self.t.float64, device=self.tensor_device)
        _lib.call("sp_gemm_exact_levels", int(ta), M, N, K, a.data_ptr(), a.stride(0), ea.data_ptr(), b.data_ptr(),
                  b.stride(0), eb.data_ptr(), bits, nsl, lv.data_ptr(), self._s())
        return lv

    def dd_levels(self, lv, nsl, tail):
        _, M, N = lv.shape
        hi = self.t.empty((M, N), dtype=self.t.float64, device=self.tensor_device)
        lo = self.t.empty_like(hi)
        _lib.call("sp_dd_levels", M, N, lv.data_ptr(), nsl, None if tail is None else tail.data_ptr(), hi.data_ptr(),
                  lo.data_ptr(), N, self._s())
        return hi, lo

    def exact_mm(self, ta, a_hi, a_lo, b, b_lo):
        """(a_hi + a_lo)(b + b_lo) for A, B double-doubles (ta = 0 only): the
        product W E of the sharded enrichment, returned as a double-double."""
        assert ta == 0
        M, K = a_hi.shape
        N = b.shape[1]
        # op(A) B with A = W (dd): W_hi (B_hi + B_lo) nearly exact + W_lo B
        hi = self.t.empty((M, N), dtype=self.t.float64, device=self.tensor_device)
        lo = self.t.empty_like(hi)
        b = b.contiguous()
        _lib.call("sp_gemm_exact", 0, M, N, K, a_hi.data_ptr(), K, b.data_ptr(),
                  None if b_lo is None else b_lo.data_ptr(), N, hi.data_ptr(), lo.data_ptr(), N, self._s())
        tail = self.t.empty_like(hi)
        _lib.call("sp_gemm", 0, 0, M, N, K, 1.0, a_lo.data_ptr(), K, b.data_ptr(), N, 0.0, tail.data_ptr(), N,
                  self._s())
        # (hi, lo) += tail: one more double-double level
        lv = self.t.stack([hi, lo + tail])
        return self.dd_levels(lv, 2, None)

    def svd_full(self, x):
        from .kernels import thin_svd
        f = thin_svd(x.contiguous())
        return f.u, f.s, f.v

    def check_finite(self, x, msg):
        from .errors import NumericalError
        if not bool(self.t.isfinite(x).all()):
            raise NumericalError(msg)

    class _PqdState:
        pass

    def pqd_state(self, e_i, k):
        m, n_i = e_i.shape
        st = self._PqdState()
        st.m, st.len, st.k = m, n_i, k
        f64 = dict(dtype=self.t.float64, device=self.tensor_device)
        st.wk = self.t.empty((m, max(n_i, 1)), **f64)
        st.qt = self.t.zeros((k, max(n_i, 1)), **f64)
        st.r = self.t.empty((k, m), **f64)
        st.perm = self.t.empty((m,), dtype=self.t.int64, device=self.tensor_device)
        st.pn2 = self.t.empty((m,), **f64)
        st.delta = self.t.zeros((max(k, 1),), **f64)
        st.part2 = self.t.empty((1,), **f64)
        st.coef = self.t.zeros((m,), **f64)
        st.jsel = self.t.empty((1,), dtype=self.t.int64, device=self.tensor_device)
        st.status = self.t.zeros((1,), dtype=self.t.int32, device=self.tensor_device)
        e_i = e_i.contiguous()
        _lib.call("sp_pqd_begin", m, n_i, k, e_i.data_ptr(), max(n_i, 1), st.wk.data_ptr(), st.perm.data_ptr(),
                  st.r.data_ptr(), m, st.pn2.data_ptr(), self._s())
        return st

    def pqd_select(self, st, t, n2):
        _lib.call("sp_pqd_select", t, st.k, st.m, st.len, n2.data_ptr(), st.perm.data_ptr(), st.r.data_ptr(), st.m,
                  st.wk.data_ptr(), st.qt.data_ptr(), st.delta.data_ptr(), st.jsel.data_ptr(), self._s())
        return st.delta[:t]

    def pqd_orth(self, st, t, delta):
        d = delta if t > 0 else st.delta
        _lib.call("sp_pqd_orth", t, st.len, d.data_ptr(), st.r.data_ptr(), st.m, st.wk.data_ptr(), st.qt.data_ptr(),
                  st.part2.data_ptr(), self._s())
        return st.part2

    def pqd_coef(self, st, t, part2):
        _lib.call("sp_pqd_coef", t, st.m, st.len, part2.data_ptr(), st.r.data_ptr(), st.m, st.wk.data_ptr(),
                  st.qt.data_ptr(), st.coef.data_ptr(), st.status.data_ptr(), self._s())
        return st.coef

    def pqd_update(self, st, t, coef):
        _lib.call("sp_pqd_update", t, st.m, st.len, coef.data_ptr(), st.r.data_ptr(), st.m, st.wk.data_ptr(),
                  st.qt.data_ptr(), st.pn2.data_ptr(), self._s())
        return st.pn2

    def pqd_check(self, st):
        from .errors import NumericalError
        if int(st.status.item()) != 0:
            raise NumericalError("sharded pivoted QR: exactly zero pivot (the deterministic filler of "
                                 "src/kernels.py:145-155 needs the unsharded candidates)")

    def id_from_qr(self, perm, rr, k):
        m = perm.shape[0]
        p = self.t.empty((m, k), dtype=self.t.float64, device=self.tensor_device)
        ind = self.t.empty((k,), dtype=self.t.int64, device=self.tensor_device)
        info = _lib.new_info()
        _lib.call("sp_id_from_qr", m, k, perm.data_ptr(), rr.data_ptr(), m, p.data_ptr(), ind.data_ptr(),
                  _lib.info_ptr(info), self._s())
        return p, ind, bool(info[_lib.INFO_WARN] & _lib.SP_WARN_ID_PINV)

    def take_rows(self, x, ind):
        return x.index_select(0, ind).contiguous() if x.shape[1] else x[:ind.shape[0]]

    def scale_cols(self, x, d):
        dd = self.t.from_numpy(np.ascontiguousarray(d)).to(self.tensor_device)
        _lib.call("sp_scale_columns", x.shape[0], x.shape[1], x.data_ptr(), x.stride(0), dd.data_ptr(), 0, self._s())
        return x

    def atz_t(self, a, z):
        """z^T a for an FP32 a (the TMA A pass widens in registers), r x n."""
        return self.atz(a, z).t().contiguous()

    def complete_other(self, x, r, k, kp):
        if r > 0:
            _lib.call("sp_gemm", 0, 0, x.shape[0], k - r, r, -1.0, x.data_ptr(), x.stride(0), kp.data_ptr(), k - r,
                      0.0, x[:, r:].data_ptr(), x.stride(0), self._s())
        return x


def _sharded_enrichment(c_i, q, n_c, comm, ops):
    """E_i = (C C^T)^q C_i, column-sharded like C, with no rank repeating
    another's products: W = sum_i C_i C_i^T is formed from nearly exact
    per-rank level products (Ozaki slices on DMMA, csrc/exact_gemm.cu) on a
    slicing grid common to all ranks (allreduce-max of the row exponents), so
    the allreduce-sum of the levels is EXACT; then E_i = W C_i locally, nearly
    exactly rounded with W in double-double.  In exact arithmetic this is the
    reference's C (C^T C) (src/power.py:282-285); computed this close to it,
    the greedy pivots downstream are the exact product's."""
    if q == 0:
        return c_i
    e_rows = comm.allreduce_max(ops.exponents(c_i, axis=1), ops)       # per row of C (m)
    bits, nsl = ops.exact_plan(n_c)
    ct = ops.transpose(c_i)                                             # n_ci x m: B = C_i^T
    lv = comm.allreduce_sum(ops.exact_levels(0, c_i, e_rows, ct, e_rows, bits, nsl), ops)
    w_hi, w_lo = ops.dd_levels(lv, nsl, None)
    e = c_i
    lo = None
    for _ in range(q):
        e, lo = ops.exact_mm(0, w_hi, w_lo, e, lo)   # (W_hi + W_lo)(E + E_lo)
    ops.check_finite(e, "power iterate overflowed; enable re-orthonormalization (reorth)")
    return e


def distributed_pivoted_qr(e_i, k: int, comm, ops):
    """Greedy column-pivoted QR of E^T (src/kernels.py:97-142) where the
    candidates are the m rows of E and every candidate is sharded across the
    ranks (E_i: m x n_ci): per step the partial norms, re-orthogonalisation
    dots, pivot norm and update coefficients are allreduce-summed (m, t, 1, m
    values).  Returns (perm (m), R (k x m)) -- the same
    on every rank."""
    m, n_i = e_i.shape
    st = ops.pqd_state(e_i, k)
    pn2 = st.pn2
    for t in range(k):
        n2 = comm.allreduce_sum(pn2, ops)
        delta = ops.pqd_select(st, t, n2)
        if t > 0:
            delta = comm.allreduce_sum(delta, ops)
        part2 = comm.allreduce_sum(ops.pqd_orth(st, t, delta), ops)
        coef = ops.pqd_coef(st, t, part2)
        if t + 1 < m:
            coef = comm.allreduce_sum(coef, ops)
            pn2 = ops.pqd_update(st, t, coef)
    ops.pqd_check(st)
    return st.perm, st.r


def sharded_power_id(a_local, c_begin: int, cols, k: int, q: int, comm, ops, r=None, n_total=None):
    """Rank-local part of the column-sharded single-pass power ID (SURVEY.md
    8(e) item 5, the per-step-allreduce variant; src/power.py:252-308 with an
    injection sketch at the column set, the BASELINE case s0 == A(:, I)).

    Rank i gathers its coarse columns C_i locally; the enrichment E_i (column
    slab of C C^T C) and the greedy pivoted QR of E^T are distributed with
    sketch-sized allreduces only; P and the pivots come out identical on every
    rank.  The lifting T = (V_r S_r^-1)(U_r^T A) stays factored and sharded:
    U_r, S_r, V_r,i from the distributed range finder (no gather of C), the
    left factor's rows V_r,i S_r^-1 for this rank's coarse columns, the right
    factor's columns U_r^T A_i for its slab.

    Returns (P m x k, indices k, skeleton_i k x n_ci, left_i n_ci x r,
    right_i r x n_i, r): P / indices replicated; skeleton and left row-blocks
    of the coarse index order (rank order = global order: I is ascending and
    the slabs are contiguous)."""
    cols = _validate_cols(cols, k, n_total)
    m, n_i = a_local.shape
    sel = (cols >= c_begin) & (cols < c_begin + n_i)
    c_i = ops.gather(a_local, cols[sel] - c_begin)
    n_c = cols.size
    if k > min(m, n_c):
        from .errors import ConfigError
        raise ConfigError(f"rank k={k} outside [1, {min(m, n_c)}]")
    e_i = _sharded_enrichment(c_i, q, n_c, comm, ops)
    perm, rr = distributed_pivoted_qr(e_i, k, comm, ops)
    p, ind, warn = ops.id_from_qr(perm, rr, k)
    if warn:
        import warnings as _w
        from .errors import RankDeficiencyWarning
        _w.warn("ID pivots are rank deficient; using pseudo-inverse solve", RankDeficiencyWarning, stacklevel=2)
    skel_i = ops.take_rows(c_i, ind)
    # lifting rank r = max(k, min(2k, rank)) clamped to the rank (src/rowid.py:130-134)
    r_req = int(r) if r is not None else 0
    row0 = int(np.count_nonzero(cols < c_begin))
    need = max(2 * k, r_req)
    u, s_c, rank, v_i = distributed_sketch_basis(c_i, row0, n_c, 1.0, comm, ops, need=need, want_v=True)
    r_use = r_req if r_req else max(k, min(2 * k, rank))
    if r_use > rank:
        import warnings as _w
        from .errors import RankDeficiencyWarning
        _w.warn(f"lifting rank {r_use} clamped to sketch rank {rank}", RankDeficiencyWarning, stacklevel=2)
        r_use = rank
    ur = ops.cols(u, 0, r_use)
    inv = 1.0 / np.asarray(s_c[:r_use], dtype=np.float64)
    left_i = ops.scale_cols(ops.cols(v_i, 0, r_use), inv)               # V_r,i S_r^-1
    right_i = ops.matmul_tn(ur, ops.contig(a_local)) if a_local.dtype.itemsize == 8 else ops.atz_t(a_local, ur)
    return p, ind, skel_i, left_i, right_i, r_use


def shard_columns(n: int, world: int, rank: int, align: int = 1) -> tuple[int, int]:
    """Contiguous column slab of a rank (rounded to ``align`` columns)."""
    units = n // align
    b = (units * rank // world) * align
    e = (units * (rank + 1) // world) * align if rank + 1 < world else n
    return b, e

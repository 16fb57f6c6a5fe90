"""Column-sharded power SVD on CPU: world_size 2 over gloo, the exchange
logic of paper_2105_01271_b200.sharded driven with a numpy arithmetic
backend (test infrastructure), checked against the single-process target
and against world_size 1."""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


class NumpyOps:
    """CPU stand-in for DeviceOps (float64 torch CPU tensors, LAPACK math)."""

    tensor_device = torch.device("cpu")

    def _t(self, a):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))

    def zeros(self, shape):
        return torch.zeros(shape, dtype=torch.float64)

    def empty_like(self, x):
        return torch.empty_like(x)

    def contig(self, x):
        return x.contiguous()

    def pad_cols(self, x, w):
        out = self.zeros((x.shape[0], w))
        out[:, :x.shape[1]] = x
        return out

    def cat_cols(self, parts):
        return torch.cat(parts, 1).contiguous()

    def cat_rows(self, parts):
        return torch.cat(parts, 0).contiguous()

    def rows(self, x, a, b):
        return x[a:b].contiguous()

    def cols(self, x, a, b):
        return x[:, a:b].contiguous()

    def set_cols(self, x, blk, c0):
        x[:, c0:c0 + blk.shape[1]] = blk
        return x

    def to_numpy(self, x):
        return x.numpy()

    def gather(self, a, idx):
        return self._t(a.numpy()[:, idx])

    def pad_rows(self, x, r):
        if x.shape[0] >= r:
            return x
        out = self.zeros((r, x.shape[1]))
        out[:x.shape[0]] = x
        return out

    def fill_uniform(self, rows, cols, seed, row0):
        # the device counter-based hash (csrc/common.cuh hash_uniform) on the global index
        with np.errstate(over="ignore"):
            i = (np.arange(rows * cols, dtype=np.uint64) + np.uint64(row0 * cols))
            z = (np.uint64(seed) * np.uint64(0x9E3779B97F4A7C15) + i * np.uint64(0xD1B54A32D192ED03)
                 + np.uint64(0x8CB92BA72F3D8DD7))
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z ^= z >> np.uint64(31)
        u = (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0) * 2.0 - 1.0
        return self._t(u.reshape(rows, cols))

    def matmul_tn(self, a, b):
        return self._t(a.numpy().T @ b.numpy())

    def tsqr(self, x):
        return self.qr(x, False)

    def new_flag(self):
        return torch.zeros((1,), dtype=torch.float64)

    def flag_value(self, flag):
        return flag.clone()

    def qr_async(self, x, flag):
        return self.qr(x, True)

    def svd_small_t(self, m):
        u, s, _ = np.linalg.svd(m.numpy().T)
        return self._t(u), self._t(s)

    def sketch_basis(self, c, power):
        u, s, _ = np.linalg.svd(c.numpy(), full_matrices=False)
        r = int(np.count_nonzero((s / s[0]) ** power > 1e-12)) if s[0] > 0 else 0
        return self._t(u[:, :r]), s[:r], r

    def atz(self, a, z):
        return self._t(a.numpy().T @ z.numpy())

    def qr(self, x, well_conditioned):
        q, r = np.linalg.qr(x.numpy())
        sg = np.where(np.diag(r) < 0, -1.0, 1.0)
        return self._t(q * sg), self._t(r * sg[:, None])

    def matmul(self, a, b):
        return self._t(a.numpy() @ b.numpy())

    def svd_small(self, m):
        u, s, vt = np.linalg.svd(m.numpy())
        return self._t(u), self._t(s), self._t(vt.T)

    def _hh(self, q, r, k):
        # Householder reconstruction: LU of Q - [S; 0] (csrc/complete.cu)
        w = q[:k, :r].copy()
        sgn = np.zeros(r)
        lmat = np.zeros((k, r))
        umat = np.zeros((r, r))
        for i in range(r):
            sgn[i] = -1.0 if w[i, i] >= 0 else 1.0
            w[i, i] -= sgn[i]
            umat[i, i:] = w[i, i:]
            lmat[i:, i] = w[i:, i] / w[i, i]
            w[i + 1:, i + 1:] -= np.outer(lmat[i + 1:, i], umat[i, i + 1:])
        ui = np.linalg.inv(umat)
        t = -umat @ np.diag(sgn) @ np.linalg.inv(lmat[:r]).T
        kp = ui @ t @ ui.T @ q[r:k, :r].T
        etop = np.zeros((k, k - r))
        etop[:r] = sgn[:, None] * kp
        etop[r:] = np.eye(k - r)
        return kp, etop

    def complete(self, x, r, k):
        q = x.numpy()
        if r == 0:
            q[:, :] = 0.0
            q[:k, :k] = np.eye(k)
            return x
        kp, etop = self._hh(q, r, k)
        q[:, r:] = -q[:, :r] @ kp
        q[:k, r:] += etop
        return x

    def complete_root(self, x, r, k):
        q = x.numpy()
        if r == 0:
            return self.complete(x, r, k), self.zeros((0, k))
        kp, _ = self._hh(q, r, k)
        self.complete(x, r, k)
        return x, self._t(kp)

    def complete_other(self, x, r, k, kp):
        q = x.numpy()
        if r > 0:
            q[:, r:] = -q[:, :r] @ kp.numpy()
        return x

    # --- the sharded ID: numpy emulation of the device entry points (same
    # slicing grids, exact level products, per-step partial sums)
    BITS_PLAN = None

    def exponents(self, x, axis):
        mx = np.abs(x.numpy()).max(axis=axis)
        _, e = np.frexp(mx)
        return torch.from_numpy(np.where(mx > 0, e, -100000).astype(np.int32))

    def exact_plan(self, K):
        return int(np.floor((53 - np.ceil(np.log2(max(K, 1)))) / 2)), 2

    @staticmethod
    def _head(x, e, bits, axis):
        ee = np.expand_dims(e.astype(np.float64), axis)
        unit = np.exp2(ee - bits)
        h = np.where(ee < -90000, 0.0, np.trunc(x / unit) * unit)
        return h, x - h

    def transpose(self, x):
        return x.t().contiguous()

    def exact_levels(self, ta, a, ea, b, eb, bits, nsl):
        a_ = a.numpy().T if ta else a.numpy()
        s0, s1 = self._head(a_, ea.numpy(), bits, 1)
        t0, t1 = self._head(b.numpy(), eb.numpy(), bits, 0)
        return self._t(np.stack([s0 @ t0, s0 @ t1 + s1 @ b.numpy()]))

    def dd_levels(self, lv, nsl, tail):
        lv = lv.numpy()
        s, err = lv[0].copy(), np.zeros_like(lv[0])
        for L in range(1, nsl):
            x = lv[L]
            t = s + x
            bb = t - s
            err += (s - (t - bb)) + (x - bb)
            s = t
        if tail is not None:
            err += tail.numpy()
        h = s + err
        return self._t(h), self._t(err - (h - s))

    def exact_mm(self, ta, a_hi, a_lo, b, b_lo):
        bits, nsl = self.exact_plan(a_hi.shape[1])
        e_a = self.exponents(a_hi, 1)
        e_b = self.exponents(b, 0)
        lv = self.exact_levels(0, a_hi, e_a, b, e_b, bits, nsl)
        tail = a_hi.numpy() @ b_lo.numpy() if b_lo is not None else 0.0
        tail = tail + a_lo.numpy() @ b.numpy()
        return self.dd_levels(lv, nsl, self._t(tail))

    def svd_full(self, x):
        u, sv, vt = np.linalg.svd(x.numpy(), full_matrices=False)
        return self._t(u), self._t(sv), self._t(vt.T)

    def check_finite(self, x, msg):
        assert np.all(np.isfinite(x.numpy())), msg

    class _St:
        pass

    def pqd_state(self, e_i, k):
        st = self._St()
        st.w = e_i.numpy().copy()                 # candidate j = row j (local entries)
        st.m, st.len, st.k = st.w.shape[0], st.w.shape[1], k
        st.qt = np.zeros((k, st.len))
        st.r_np = np.zeros((k, st.m))
        st.perm_np = np.arange(st.m)
        st.pn2 = self._t((st.w * st.w).sum(axis=1))
        return st

    def pqd_select(self, st, t, n2):
        nrm = np.sqrt(n2.numpy())
        cand = t + np.flatnonzero(nrm[t:] == nrm[t:].max())
        j = cand[np.argmin(st.perm_np[cand])]
        if j != t:
            st.w[[t, j]] = st.w[[j, t]]
            st.r_np[:, [t, j]] = st.r_np[:, [j, t]]
            st.perm_np[[t, j]] = st.perm_np[[j, t]]
        return self._t(st.qt[:t] @ st.w[t])

    def pqd_orth(self, st, t, delta):
        d = delta.numpy()
        st.r_np[:t, t] += d
        st.qt[t] = st.w[t] - d @ st.qt[:t]
        return self._t(np.array([st.qt[t] @ st.qt[t]]))

    def pqd_coef(self, st, t, part2):
        pn = np.sqrt(part2.numpy()[0])
        st.r_np[t, t] = pn
        assert pn > 0
        st.qt[t] = st.qt[t] / pn
        coef = np.zeros(st.m)
        coef[t + 1:] = st.w[t + 1:] @ st.qt[t]
        return self._t(coef)

    def pqd_update(self, st, t, coef):
        c = coef.numpy()
        st.r_np[t, t + 1:] = c[t + 1:]
        st.w[t + 1:] -= np.outer(c[t + 1:], st.qt[t])
        return self._t((st.w * st.w).sum(axis=1))

    def pqd_check(self, st):
        st.perm = torch.from_numpy(st.perm_np.copy())
        st.r = self._t(st.r_np)

    def id_from_qr(self, perm, rr, k):
        from scipy.linalg import solve_triangular
        perm, r = perm.numpy(), rr.numpy()
        m = perm.size
        coef = solve_triangular(r[:, :k], r[:, k:])
        p = np.zeros((m, k))
        p[perm[:k]] = np.eye(k)
        p[perm[k:]] = coef.T
        return self._t(p), torch.from_numpy(perm[:k].copy()), False

    def take_rows(self, x, ind):
        return self._t(x.numpy()[ind.numpy()])

    def scale_cols(self, x, d):
        return self._t(x.numpy() * d[None, :])

def _field(noisy=False):
    from paper_2105_01271_b200.datagen import CONFIGS, FieldConfig, coarse_grid_indices, generate_host
    if noisy:
        # a noise floor just below the kept-rank cut (the cfg3 regime): the range
        # finder needs several subspace steps -- Rayleigh-Ritz steps with blind
        # steps in between, the same number on every rank
        cfg = FieldConfig("shard_noisy", 300, (48, 64), 20, 0.5, 0.001, 2, 4, 30, 1, noise_std=1e-4)
    else:
        cfg = CONFIGS["cfg2"].scaled(m=300, grid=(48, 64), name="shard")
    return cfg, generate_host(cfg), coarse_grid_indices(cfg.grid, cfg.stride)


def _worker(rank, world, port, out_q, noisy=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2105_01271_b200.sharded import TorchComm, shard_columns, sharded_power_svd
    cfg, a, cols = _field(noisy)
    b, e = shard_columns(cfg.n, world, rank, align=cfg.grid[1])  # x-slabs of the grid
    ops = NumpyOps()
    u, s, v, r, warn = sharded_power_svd(torch.from_numpy(a[:, b:e].copy()), b, cols, 30, 1, TorchComm(), ops)
    parts = [None] * world
    dist.all_gather_object(parts, (b, e, v.numpy()))
    if rank == 0:
        out_q.put((u.numpy(), s, np.concatenate([p[2] for p in sorted(parts, key=lambda t: t[0])]), r, warn))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [1, 2])
def test_sharded_matches_target(world):
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(rk, world, port, q)) for rk in range(world)]
    for p in procs:
        p.start()
    u, s, v, r, warn = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg, a, cols = _field()
    tu, ts, tv, tr = oracle.projector_target_svd(a, a[:, cols], 30, 3)
    assert r == tr and warn
    np.testing.assert_allclose(s[:r], ts, rtol=0, atol=1e-12 * ts[0])
    assert np.all(s[r:] == 0)
    np.testing.assert_allclose(u.T @ u, np.eye(30), atol=1e-12)
    np.testing.assert_allclose(v.T @ v, np.eye(30), atol=1e-12)
    rec = (u * s) @ v.T
    np.testing.assert_allclose(rec, (tu * ts) @ tv.T, atol=1e-10 * np.abs(a).max())


@pytest.mark.parametrize("world", [1, 2])
def test_sharded_noisy_field_blind_steps(world):
    """Several subspace steps (a noise bulk right below the kept-rank cut):
    blind steps between the Rayleigh-Ritz steps, identical on every rank (no
    collective mismatch), result against the dense target."""
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(rk, world, port, q, True)) for rk in range(world)]
    for p in procs:
        p.start()
    u, s, v, r, warn = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg, a, cols = _field(True)
    tu, ts, tv, tr = oracle.projector_target_svd(a, a[:, cols], 30, 3)
    assert r == tr
    np.testing.assert_allclose(s[:r], ts, rtol=0, atol=1e-12 * ts[0])
    assert oracle.principal_angle(u[:, :r], tu) <= 1e-8


def _id_field():
    """A field whose 20 ID pivots are gap-determined: a slow-decay random
    block (the tests/golden/id_slow.npz construction) -- the per-rank partial
    sums may not disturb the greedy selection."""
    import sys as _s
    _s.path.insert(0, str(ROOT / "tests"))
    from conftest import philox, rank_deficient
    a = rank_deficient(philox(41), 160, 1536, rank=60, decay=np.logspace(0, -1, 60))
    return a, np.arange(0, 1536, 6)


def _id_worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2105_01271_b200.sharded import TorchComm, shard_columns, sharded_power_id
    a, cols = _id_field()
    b, e = shard_columns(a.shape[1], world, rank, align=48)
    p, ind, skel, left, right, r = sharded_power_id(torch.from_numpy(a[:, b:e].copy()), b, cols, 20, 1,
                                                    TorchComm(), NumpyOps(), n_total=a.shape[1])
    parts = [None] * world
    dist.all_gather_object(parts, (b, p.numpy(), ind.numpy(), skel.numpy(), left.numpy(), right.numpy()))
    if rank == 0:
        out_q.put((parts, r))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2, 4])
def test_sharded_power_id_matches_single_process(world):
    # the per-step-allreduce variant of the column-sharded ID (SURVEY 8(e)
    # item 5): enrichment from exact level products allreduce-summed, the
    # pivoted QR's norms / dots / coefficients allreduce-summed each step;
    # P and the pivots replicated bit-for-bit; skeleton and the lifting's
    # factors sharded.  Against the oracle's power_id algebra.
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_id_worker, args=(rk, world, port, q)) for rk in range(world)]
    for p in procs:
        p.start()
    parts, r = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    parts = sorted(parts, key=lambda t: t[0])
    for other in parts[1:]:  # replicated parts: identical bits on every rank
        for x, y in zip(parts[0][1:3], other[1:3]):
            assert np.array_equal(x, y)
    a, cols = _id_field()
    idx, w = cols[None, :], np.ones((1, cols.size))
    ref = oracle.spc_power_id(a, idx, w, cols, 20, q=1)
    assert np.all(ref.pivot_gaps > 1e-11)
    _, pp, ind, _, _, _ = parts[0]
    assert np.array_equal(ind, ref.indices)
    np.testing.assert_allclose(pp, ref.p, rtol=0, atol=1e-10 * np.abs(ref.p).max())
    skel = np.concatenate([t[3] for t in parts], axis=1)
    assert np.array_equal(skel, ref.skeleton)
    assert r == ref.r
    # lifting: [left_0; left_1; ..] @ [right_0 | right_1 | ...] is
    # (V_r S_r^-1)(U_r^T A), the exact-arithmetic value of build_lifting
    left = np.concatenate([t[4] for t in parts], axis=0)
    right = np.concatenate([t[5] for t in parts], axis=1)
    u, sv, v = oracle.svd_thin(a[:, cols])
    want = (v[:, :r] / sv[:r]) @ (u[:, :r].T @ a)
    np.testing.assert_allclose(left @ right, want, rtol=0, atol=1e-9 * np.abs(want).max())


def test_sharded_drivers_validate_the_column_set():
    # out-of-range / repeated / unsorted I must raise, not be
    # silently dropped or permuted by the per-shard gather
    from paper_2105_01271_b200.errors import ConfigError
    from paper_2105_01271_b200.sharded import sharded_power_id, sharded_power_svd

    class _Comm:
        rank, world = 0, 1

    a = torch.from_numpy(np.random.default_rng(0).standard_normal((12, 40)))
    for bad, msg in (([0, 5, 5, 9, 13], "distinct"), ([0, 9, 5, 13, 20], "ascending"),
                     ([0, 5, 9, 13, 40], "out of range"), ([-1, 5, 9, 13, 20], "out of range"),
                     ([0, 5], "exceed target rank")):
        for fn in (sharded_power_svd, sharded_power_id):
            with pytest.raises(ConfigError, match=msg):
                fn(a, 0, bad, 2, 1, _Comm(), NumpyOps(), n_total=40)

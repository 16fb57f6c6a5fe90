"""Column-sharded driver on the device kernels (DeviceOps).  One GPU only:
world 1 through TorchComm, and two shards emulated by two host threads that
exchange device tensors through a host-side barrier (no kernel ever waits on
another, so sharing one GPU is safe)."""

import threading
import warnings

import numpy as np
import pytest

import oracle
import paper_2105_01271_b200 as sp
from paper_2105_01271_b200.datagen import CONFIGS, generate_host
from paper_2105_01271_b200.sharded import DeviceOps, TorchComm, shard_columns, sharded_power_id, sharded_power_svd

pytestmark = pytest.mark.gpu


class ThreadComm:
    def __init__(self, rank, world, shared):
        self.rank, self.world, self.sh = rank, world, shared

    def _exchange(self, x):
        self.sh["slots"][self.rank] = x
        self.sh["bar"].wait()
        parts = list(self.sh["slots"])
        self.sh["bar"].wait()
        return parts

    def allgather_cols(self, x, ops, widths=None):
        return ops.cat_cols(self._exchange(x))

    def allgather_rows(self, x, ops):
        return ops.cat_rows(self._exchange(ops.contig(x)))

    def allreduce_sum(self, x, ops):
        parts = self._exchange(ops.contig(x))
        total = parts[0].clone()
        for p in parts[1:]:  # rank order: the same bits on every rank
            total += p
        return total

    def allreduce_max(self, x, ops):
        parts = self._exchange(ops.contig(x))
        total = parts[0].clone()
        for p in parts[1:]:
            total = total.maximum(p)
        return total

    def broadcast(self, x, root, ops):
        return self._exchange(x)[root].clone()


def _case():
    cfg = CONFIGS["cfg2"].scaled(m=400, grid=(64, 64), name="shard")
    a = generate_host(cfg)
    op, cols = sp.grid_injection(cfg.grid, cfg.stride)
    return cfg, a, op, cols


def test_world1_equals_power_svd(cuda):
    cfg, a, op, cols = _case()
    ops = DeviceOps()
    ad = cuda.from_numpy(a).cuda()
    u, s, v, r, warn = sharded_power_svd(ad, 0, cols, 50, 1, TorchComm(), ops)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        ref = sp.power_svd(sp.ArraySnapshotStream(a), op, 50, sp.PowerConfig(q=1, columns=cols))
    assert r == ref.kept_rank and warn
    np.testing.assert_allclose(s, ref.s, rtol=0, atol=1e-13 * ref.s[0])
    vh = v.cpu().numpy()
    np.testing.assert_allclose(vh.T @ vh, np.eye(50), atol=1e-12)


def test_two_shards_match_target(cuda):
    cfg, a, op, cols = _case()
    world = 2
    shared = {"slots": [None] * world, "bar": threading.Barrier(world)}
    results = [None] * world
    errors = []

    def run(rank):
        try:
            cuda.cuda.set_device(0)
            b, e = shard_columns(cfg.n, world, rank, align=cfg.grid[1])
            ad = cuda.from_numpy(a[:, b:e].copy()).cuda()
            results[rank] = (b,) + sharded_power_svd(ad, b, cols, 50, 1, ThreadComm(rank, world, shared), DeviceOps())
        except Exception as exc:  # surface in the main thread
            errors.append(exc)
            shared["bar"].abort()

    th = [threading.Thread(target=run, args=(rk,)) for rk in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errors, errors
    u = results[0][1].cpu().numpy()
    s = results[0][2]
    v = np.concatenate([results[rk][3].cpu().numpy() for rk in range(world)])
    r = results[0][4]
    assert np.array_equal(results[1][1].cpu().numpy(), u)  # replicated, bitwise identical
    tu, ts, tv, tr = oracle.projector_target_svd(a, a[:, cols], 50, 3)
    assert r == tr
    np.testing.assert_allclose(s[:r], ts, rtol=0, atol=1e-12 * ts[0])
    np.testing.assert_allclose(v.T @ v, np.eye(50), atol=1e-12)
    np.testing.assert_allclose(u.T @ u, np.eye(50), atol=1e-12)
    np.testing.assert_allclose((u * s) @ v.T, (tu * ts) @ tv.T, atol=1e-10 * np.abs(a).max())


def test_two_shards_noisy_field_blind_steps(cuda):
    """A noise bulk right below the kept-rank cut (the cfg3 regime): several
    subspace steps, Rayleigh-Ritz steps with blind steps in between -- the same
    sequence of exchanges on both shards, U bitwise identical, result against
    the dense target."""
    from paper_2105_01271_b200.datagen import FieldConfig
    cfg = FieldConfig("shard_noisy", 600, (64, 64), 20, 0.5, 0.001, 2, 4, 30, 1, noise_std=1e-4)
    a = generate_host(cfg)
    op, cols = sp.grid_injection(cfg.grid, cfg.stride)
    world = 2
    shared = {"slots": [None] * world, "bar": threading.Barrier(world, timeout=120)}
    results = [None] * world
    errors = []

    def run(rank):
        try:
            cuda.cuda.set_device(0)
            b, e = shard_columns(cfg.n, world, rank, align=cfg.grid[1])
            ad = cuda.from_numpy(a[:, b:e].copy()).cuda()
            results[rank] = (b,) + sharded_power_svd(ad, b, cols, 30, 1, ThreadComm(rank, world, shared), DeviceOps())
        except Exception as exc:  # surface in the main thread
            errors.append(exc)
            shared["bar"].abort()

    th = [threading.Thread(target=run, args=(rk,), daemon=True) for rk in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errors, errors
    assert all(r is not None for r in results)
    u = results[0][1].cpu().numpy()
    s, r = results[0][2], results[0][4]
    assert np.array_equal(results[1][1].cpu().numpy(), u)
    tu, ts, tv, tr = oracle.projector_target_svd(a, a[:, cols], 30, 3)
    assert r == tr
    np.testing.assert_allclose(s[:r], ts, rtol=0, atol=1e-12 * ts[0])
    assert oracle.principal_angle(u[:, :r], tu) <= 1e-8


def _id_case():
    """20 gap-determined ID pivots (a slow-decay block, tests/golden/id_slow.npz
    construction): the per-rank partial sums may not move the selection."""
    from conftest import philox, rank_deficient
    a = rank_deficient(philox(41), 300, 3072, rank=80, decay=np.logspace(0, -1, 80))
    return a, np.arange(0, 3072, 12)


@pytest.mark.parametrize("world", [1, 2, 3])
def test_sharded_power_id_matches_oracle(cuda, world):
    # per-step-allreduce variant of the column-sharded ID: exact enrichment
    # levels allreduce-summed, the pivoted QR's partial sums allreduce-summed
    # (pivqr_dist.cu); P and the pivots bitwise identical on every shard and
    # equal to the oracle's (all 20 gap-determined); skeleton and the lifting
    # factors sharded and assembled
    a, cols = _id_case()
    n = a.shape[1]
    k = 20
    shared = {"slots": [None] * world, "bar": threading.Barrier(world)}
    results = [None] * world
    errors = []

    def run(rank):
        try:
            cuda.cuda.set_device(0)
            b, e = shard_columns(n, world, rank, align=96)
            ad = cuda.from_numpy(a[:, b:e].copy()).cuda()
            comm = ThreadComm(rank, world, shared) if world > 1 else TorchComm()
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                out = sharded_power_id(ad, b, cols, k, 1, comm, DeviceOps(), n_total=n)
            cuda.cuda.synchronize()
            results[rank] = (b,) + tuple(x.cpu().numpy() if hasattr(x, "cpu") else x for x in out)
        except Exception as exc:  # surface in the main thread
            errors.append(exc)
            shared["bar"].abort()

    th = [threading.Thread(target=run, args=(rk,)) for rk in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errors, errors
    for other in results[1:]:
        for x, y in zip(results[0][1:3], other[1:3]):
            assert np.array_equal(x, y)
    idx, w = cols[None, :], np.ones((1, cols.size))
    ref = oracle.spc_power_id(a, idx, w, cols, k, q=1)
    assert np.all(ref.pivot_gaps > 1e-11)
    _, p, ind, _, _, _, r = results[0]
    np.testing.assert_array_equal(ind, ref.indices)
    np.testing.assert_allclose(p, ref.p, rtol=0, atol=1e-10 * np.abs(ref.p).max())
    c = a[:, cols]
    skel = np.concatenate([res[3] for res in results], axis=1)
    np.testing.assert_array_equal(skel, c[ind])
    assert r == ref.r
    left = np.concatenate([res[4] for res in results], axis=0)
    right = np.concatenate([res[5] for res in results], axis=1)
    got = left @ right
    # against the exact-arithmetic lifting (V_r S_r^-1)(U_r^T A)
    u, sv, v = oracle.svd_thin(c)
    want = (v[:, :r] / sv[:r]) @ (u[:, :r].T @ a)
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-9 * np.abs(want).max())

"""GPU stress probe: random shapes / spectra / ranks through power_svd, single_pass_svd and
power_id against the oracle's dense target of the same projector.  python scripts/fuzz_api.py [cases] [seed0]"""
import sys
import time
import warnings
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402  (checker only)
import paper_2105_01271_b200 as sp  # noqa: E402

warnings.simplefilter("ignore")
cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
bad = 0
t0 = time.time()
for seed in range(seed0, seed0 + cases):
    rng = np.random.default_rng(seed)
    m = int(rng.choice([40, 130, 300, 700, 1500, 4200, 5100]))
    n = int(rng.choice([96, 512, 3000, 8192, 20000]))
    stride = int(rng.choice([2, 3, 4, 8]))
    cols = np.arange(0, n, stride)
    nc = cols.size
    kind = rng.choice(["fast", "slow", "noisy", "lowrank", "flat"])
    r0 = int(min(m, n, rng.choice([5, 20, 60, 150])))
    u, _ = np.linalg.qr(rng.standard_normal((m, r0)))
    v, _ = np.linalg.qr(rng.standard_normal((n, r0)))
    if kind == "fast":
        s = 10.0 ** (-np.arange(r0) * rng.uniform(0.8, 2.5))
    elif kind == "slow":
        s = rng.uniform(0.55, 0.93) ** np.arange(r0)
    elif kind == "flat":
        s = np.r_[np.logspace(0, -2, min(6, r0)), np.full(max(0, r0 - 6), 3e-3)]
    else:
        s = 10.0 ** (-np.arange(r0) * 0.7)
    a = (u * s) @ v.T
    if kind == "noisy":
        a = a + 10.0 ** rng.uniform(-9, -5) * rng.standard_normal((m, n))
    q = int(rng.choice([0, 1, 1, 2]))
    kmax = min(m, nc) - 1
    if kmax < 1:
        continue
    k = int(rng.integers(1, min(kmax, 64) + 1))
    op = sp.build_sketch(sp.SketchSpec("injection", n, nc))
    if not np.array_equal(op.idx.ravel(), cols):
        cols = op.idx.ravel().copy()
    tag = f"seed {seed}: m={m} n={n} nc={nc} kind={kind} r0={r0} q={q} k={k}"
    try:
        if q == 0:
            res = sp.single_pass_svd(sp.ArraySnapshotStream(a), op, k)
        else:
            res = sp.power_svd(sp.ArraySnapshotStream(a), op, k, sp.PowerConfig(q=q, columns=cols))
        tu, ts, tv, r = oracle.projector_target_svd(a, a[:, cols], k, 2 * q + 1)
        sc = np.linalg.svd(a[:, cols], compute_uv=False)
        cut = (sc / sc[0]) ** (2 * q + 1)
        near = np.any(np.abs(np.log10(np.maximum(cut, 1e-300)) + 12.0) < 0.02)  # a sigma sits on the kept-rank cut
        ok = True
        if res.kept_rank != r and not near:
            ok = False
            print("RANK ", tag, "kept", res.kept_rank, "target", r)
        if res.kept_rank == r:
            kk = min(k, r)
            err = np.abs(res.s[:kk] - ts[:kk]).max() / ts[0] if kk else 0.0
            orth = max(np.abs(res.u.T @ res.u - np.eye(k)).max(), np.abs(res.v.T @ res.v - np.eye(k)).max())
            if err > 1e-11 or orth > 1e-9 or not np.all(np.isfinite(res.s)):
                ok = False
                print("VALUE", tag, f"sigma err {err:.2e} orth {orth:.2e}")
        if q >= 1 and seed % 3 == 0 and k <= min(m, nc) - 1:
            f = sp.power_id(sp.ArraySnapshotStream(a), op, k, sp.PowerConfig(q=q, columns=cols))
            p = np.asarray(f.p)
            ind = np.asarray(f.indices)
            if not (np.array_equal(p[ind], np.eye(k)) and len(set(ind.tolist())) == k and np.all(np.isfinite(p))):
                ok = False
                print("ID   ", tag, "contract broken")
        bad += 0 if ok else 1
    except Exception as exc:  # the reference raises on the same inputs?  report
        bad += 1
        print("EXC  ", tag, type(exc).__name__, str(exc)[:600 if cases == 1 else 160])
print(f"{cases} cases, {bad} flagged, {time.time() - t0:.0f} s")

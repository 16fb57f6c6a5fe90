"""GPU stress probe: random shapes / spectra through the dense drop-in kernels (thin_qr, thin_svd,
pivoted_qr, row_id) and the two-pass / ID entry points, against numpy and the oracle.
python scripts/fuzz_dense.py [cases] [seed0]"""
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


def spectrum(rng, p, kind):
    if kind == "graded":
        return np.logspace(0, -rng.uniform(2, 13), p)
    if kind == "flat":
        h = min(6, p)
        return np.r_[np.logspace(0, -2, h), np.full(p - h, 3e-3)]
    if kind == "equal":
        return np.ones(p)
    if kind == "lowrank":
        r = max(1, p // 3)
        return np.r_[np.linspace(2, 1, r), np.zeros(p - r)]
    return np.sort(rng.uniform(0.1, 1.0, p))[::-1]


for seed in range(seed0, seed0 + cases):
    rng = np.random.default_rng(seed)
    rows = int(rng.choice([3, 17, 33, 64, 100, 257, 300, 700, 1500, 4100, 5200]))
    cols = int(rng.choice([2, 9, 31, 32, 33, 48, 64, 100, 130, 216, 256, 300, 520]))
    kind = str(rng.choice(["graded", "flat", "equal", "lowrank", "uniform"]))
    p = min(rows, cols)
    u, _ = np.linalg.qr(rng.standard_normal((rows, p)))
    v, _ = np.linalg.qr(rng.standard_normal((cols, p)))
    s = spectrum(rng, p, kind)
    m = (u * s) @ v.T
    nm = np.linalg.norm(m)
    tag = f"seed {seed}: {rows}x{cols} {kind}"
    ok = True
    try:
        f = sp.thin_qr(m)
        e1 = np.abs(f.q.T @ f.q - np.eye(p)).max()
        e2 = np.linalg.norm(f.q @ f.r - m) / max(nm, 1e-300)
        low = float(np.abs(np.tril(f.r, -1)).max()) if p > 1 else 0.0
        qo, ro = oracle.qr_reduced(m)     # the reference's sign rule: first significant entry of each column >= 0
        first = [f.q[np.flatnonzero(np.abs(f.q[:, j]) > 1e-12 * np.abs(f.q[:, j]).max())[0], j] for j in range(p)]
        if e1 > 1e-11 or e2 > 1e-12 or low > 0 or min(first) < 0:
            ok = False
            print("QR   ", tag, f"orth {e1:.2e} recon {e2:.2e} below-diagonal {low:.2e} min first entry {min(first):.2e}")
        g = sp.thin_svd(m)
        sr = np.linalg.svd(m, compute_uv=False)
        e3 = np.abs(g.s - sr).max() / max(sr[0], 1e-300)
        e4 = max(np.abs(g.u.T @ g.u - np.eye(p)).max(), np.abs(g.v.T @ g.v - np.eye(p)).max())
        e5 = np.linalg.norm((g.u * g.s) @ g.v.T - m) / max(nm, 1e-300)
        if e3 > 1e-12 or e4 > 1e-10 or e5 > 1e-12:
            ok = False
            eu, ev = np.abs(g.u.T @ g.u - np.eye(p)).max(), np.abs(g.v.T @ g.v - np.eye(p)).max()
            print("SVD  ", tag, f"sigma {e3:.2e} orth U {eu:.2e} V {ev:.2e} recon {e5:.2e} rank {int(np.sum(s > 0))}")
        if kind in ("graded", "uniform") and p >= 2:
            k = int(rng.integers(1, min(p, 60) + 1))
            h = sp.pivoted_qr(m, k)
            _, _, perm_o = oracle.greedy_pivoted_qr(m, k)
            gaps = oracle.pivot_gaps(m, k)
            pstar = k if np.all(gaps > 1e-10) else int(np.argmax(gaps <= 1e-10))
            if not np.array_equal(h.perm[:pstar], perm_o[:pstar]):
                ok = False
                print("PQR  ", tag, f"k={k} pivots differ inside the first {pstar}")
            rid = sp.row_id(m.T.copy() if rows < cols else m, min(k, min(m.shape) if rows >= cols else min(m.T.shape)))
            pp, ind = np.asarray(rid.p), np.asarray(rid.indices)
            if not (np.array_equal(pp[ind], np.eye(ind.size)) and np.all(np.isfinite(pp))):
                ok = False
                print("RID  ", tag, "contract broken")
    except Exception as exc:
        ok = False
        print("EXC  ", tag, type(exc).__name__, str(exc)[:300])
    bad += 0 if ok else 1
print(f"{cases} cases, {bad} flagged, {time.time() - t0:.0f} s")

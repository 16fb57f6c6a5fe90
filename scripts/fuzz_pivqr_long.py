"""GPU stress probe for the long-candidate pivoted QR (the row-block path with the lagged update, csrc/pivqr.cu:
rows >= 32768 and rows >= 8 cols): random shapes and spectra, pivots against the oracle where gap-determined,
factor contracts.  python scripts/fuzz_pivqr_long.py [cases] [seed0]"""
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
cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
bad = 0
t0 = time.time()
for seed in range(seed0, seed0 + cases):
    rng = np.random.default_rng(seed)
    rows = int(rng.choice([32768, 40001, 65536, 100003, 131072]))
    cols = int(rng.choice([8, 33, 100, 257, 500]))
    cols = min(cols, rows // 8)
    kind = str(rng.choice(["graded", "steep", "lowrank", "uniform", "noisy"]))
    p = cols
    u, _ = np.linalg.qr(rng.standard_normal((rows, p)))
    v, _ = np.linalg.qr(rng.standard_normal((cols, p)))
    if kind == "graded":
        s = np.logspace(0, -rng.uniform(2, 12), p)
    elif kind == "steep":
        s = 10.0 ** (-np.arange(p) * rng.uniform(1.0, 4.0))        # one-step drops of 1e1 .. 1e4
        s = np.maximum(s, 1e-300)
    elif kind == "lowrank":
        r = max(1, p // 4)
        s = np.r_[np.linspace(2, 1, r), np.zeros(p - r)]
    elif kind == "noisy":
        s = np.r_[np.logspace(0, -3, min(5, p)), np.full(max(0, p - 5), 1e-7)]
    else:
        s = np.sort(rng.uniform(0.1, 1.0, p))[::-1]
    m = (u * s) @ v.T
    k = int(rng.integers(1, min(p, 60) + 1))
    tag = f"seed {seed}: {rows}x{cols} {kind} k={k}"
    ok = True
    try:
        h = sp.pivoted_qr(m, k)
        q_o, r_o, perm_o = oracle.greedy_pivoted_qr(m, k)
        gaps = oracle.pivot_gaps(m, k)
        pstar = k if np.all(gaps > 1e-10) else int(np.argmax(gaps <= 1e-10))
        if not np.array_equal(h.perm[:pstar], perm_o[:pstar]):
            ok = False
            print("PQR  ", tag, f"pivots differ inside the first {pstar}: {h.perm[:pstar]} vs {perm_o[:pstar]}")
        q, r = np.asarray(h.q), np.asarray(h.r)
        e1 = np.abs(q[:, :pstar].T @ q[:, :pstar] - np.eye(pstar)).max() if pstar else 0.0
        e2 = np.linalg.norm(q[:, :pstar] @ r[:pstar] - m[:, h.perm]) if pstar else 0.0
        # the factorisation of the gap-determined prefix reproduces the oracle's
        e3 = np.abs(np.abs(r[:pstar, :pstar]) - np.abs(r_o[:pstar, :pstar])).max() / max(np.abs(r_o).max(), 1e-300) if pstar else 0.0
        if e1 > 1e-10 or e3 > 1e-9 or not np.all(np.isfinite(r)):
            ok = False
            print("PQR  ", tag, f"orth {e1:.2e} R diff {e3:.2e} (residual of the prefix {e2:.2e})")
    except Exception as exc:
        ok = False
        print("EXC  ", tag, type(exc).__name__, str(exc)[:300])
    bad += 0 if ok else 1
print(f"{cases} cases, {bad} flagged, {time.time() - t0:.0f} s")

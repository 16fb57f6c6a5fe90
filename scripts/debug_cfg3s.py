"""GPU debug probe: orthonormality of the padded factors at cfg3s."""
import sys
import warnings
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2105_01271_b200 as sp  # noqa: E402
from paper_2105_01271_b200 import _lib  # noqa: E402
from paper_2105_01271_b200.datagen import FieldConfig, generate_host  # noqa: E402

warnings.simplefilter("ignore")
cfg = FieldConfig("cfg3s", 1000, (128, 128), 40, 0.5, 0.001, 2, 8, 100, 1, noise_std=1e-4)
a = generate_host(cfg)
op, idx = sp.grid_injection(cfg.grid, cfg.stride)
for k in (20, 50, 100):
    res = sp.power_svd(sp.ArraySnapshotStream(a), op, k, sp.PowerConfig(q=1, columns=idx))
    e = np.abs(res.u.T @ res.u - np.eye(k))
    ev = np.abs(res.v.T @ res.v - np.eye(k))
    bad = np.argwhere(e > 1e-10)
    print(f"k={k} kept={res.kept_rank} maxU={e.max():.2e} maxV={ev.max():.2e} nbadU={len(bad)}",
          "first bad", bad[:5].tolist())

s = torch.cuda.current_stream().cuda_stream
rng = np.random.default_rng(0)
for (m, r, k) in [(1000, 7, 100), (1000, 7, 50), (2000, 7, 100), (1000, 0, 100), (16384, 7, 100)]:
    q0, _ = np.linalg.qr(rng.standard_normal((m, max(r, 1))))
    w = np.concatenate([q0[:, :r], rng.uniform(-1, 1, (m, k - r))], axis=1)
    dw = torch.from_numpy(np.ascontiguousarray(w)).cuda()
    q = torch.empty((m, k), dtype=torch.float64, device="cuda")
    rr = torch.empty((k, k), dtype=torch.float64, device="cuda")
    _lib.call("sp_tsqr", m, k, dw.data_ptr(), k, q.data_ptr(), k, rr.data_ptr(), k, s)
    qh = q.cpu().numpy()
    e = np.abs(qh.T @ qh - np.eye(k))
    print(f"tsqr {m}x{k} (r={r}): orth {e.max():.2e} recon {np.linalg.norm(qh @ rr.cpu().numpy() - w):.2e}",
          "bad cols", sorted(set(np.argwhere(e > 1e-10)[:, 1].tolist()))[:12])

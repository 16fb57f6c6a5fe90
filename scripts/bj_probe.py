"""GPU probe: the size-general thin_svd on wide full-rank cores (block Jacobi
path): time and accuracy against LAPACK."""
import sys, time, json
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2105_01271_b200 as sp
from threadpoolctl import threadpool_limits
out = {}
rng = np.random.default_rng(0)
for (m, n) in ((1500, 1100), (5000, 4096), (2000, 20000)):
    x = rng.standard_normal((m, n)) * np.logspace(0, -6, n)[None, :]
    xd = torch.from_numpy(x).cuda()
    sp.thin_svd(xd[:200, :150].contiguous())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = sp.thin_svd(xd)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    s = f.s.cpu().numpy()
    with threadpool_limits(16):
        st = np.linalg.svd(x, compute_uv=False)
    u, v = f.u, f.v
    p = min(m, n)
    eye = torch.eye(p, dtype=torch.float64, device="cuda")
    orth_u = float((u.T @ u - eye).abs().max())
    orth_v = float((v.T @ v - eye).abs().max())
    rec = float(((u * f.s) @ v.T - xd).abs().max()) / float(xd.abs().max())
    out[f"{m}x{n}"] = {"s": dt, "max_ds_over_s1": float(np.max(np.abs(s - st)) / st[0]),
                       "max_rel_ds_top": float(np.max(np.abs(s[:p // 2] - st[:p // 2]) / st[:p // 2])),
                       "orth_u": orth_u, "orth_v": orth_v, "rec": rec}
    print(json.dumps({f"{m}x{n}": out[f"{m}x{n}"]}), flush=True)
    del xd, f, u, v
    torch.cuda.empty_cache()

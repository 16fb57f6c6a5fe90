"""GPU probe: time (and, built with SPB_NVCC_EXTRA=-DSPB_JACOBI_TRACE, sweeps) of the
Jacobi SVD kernels on dense, graded and nearly-diagonal cores.  python scripts/jacobi_probe.py"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_01271_b200 import _lib  # noqa: E402

st = torch.cuda.current_stream()
rng = np.random.default_rng(0)
for n in (64, 120, 216, 256):
    cases = {"dense gaussian": rng.standard_normal((n, n)),
             "graded 1e-10": rng.standard_normal((n, n)) @ np.diag(np.logspace(0, -10, n)),
             "nearly diagonal (Ritz restart)": np.diag(np.linspace(1.0, 0.5, n)) + 1e-6 * rng.standard_normal((n, n)),
             "7 large + flat bulk": np.diag(np.r_[np.logspace(0, -3, 7), np.full(n - 7, 3e-5)]) @ np.linalg.qr(rng.standard_normal((n, n)))[0]}
    for name, m in cases.items():
        d = torch.from_numpy(np.ascontiguousarray(m)).cuda()
        U = torch.empty((n, n), dtype=torch.float64, device="cuda")
        V = torch.empty((n, n), dtype=torch.float64, device="cuda")
        S = torch.empty(n, dtype=torch.float64, device="cuda")
        f = lambda: _lib.call("sp_jacobi_svd", n, d.data_ptr(), n, U.data_ptr(), n, S.data_ptr(), V.data_ptr(), n, st.cuda_stream)
        f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            f()
        e1.record()
        torch.cuda.synchronize()
        s_ref = np.linalg.svd(m, compute_uv=False)
        err = np.abs(S.cpu().numpy() - s_ref).max() / s_ref[0]
        print(f"n={n:4d} {name:32s} {e0.elapsed_time(e1) / 3:8.3f} ms  sigma err {err:.1e}", flush=True)

"""GPU probe: the A pass (K2) under a sustained run -- per-launch CUDA-event
times, SM clocks and power sampled during the loop.  One variant per process
(SPB_K2_FMA=1 selects the scalar-DFMA consumers; default DMMA).

    python scripts/k2_power_probe.py [r] [launches] [m] [n] [f64|f32]
"""
import json
import statistics
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from bench import ClockSampler  # noqa: E402
from paper_2105_01271_b200 import _lib  # noqa: E402

r = int(sys.argv[1]) if len(sys.argv) > 1 else 8
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
m = int(sys.argv[3]) if len(sys.argv) > 3 else 10000
n = int(sys.argv[4]) if len(sys.argv) > 4 else 1 << 20
dt = torch.float32 if (len(sys.argv) > 5 and sys.argv[5] == "f32") else torch.float64
dev = torch.device("cuda", 0)
A = torch.empty((m, n), dtype=dt, device=dev)
for i in range(0, m, 500):
    A[i:i + 500].normal_()
Z = torch.randn((m, r), dtype=torch.float64, device=dev)
Y = torch.empty((n, r), dtype=torch.float64, device=dev)
s = torch.cuda.current_stream()
tag = _lib.SP_F64 if dt == torch.float64 else _lib.SP_F32


def apass():
    _lib.call("sp_skinny_atz", A.data_ptr(), tag, m, n, n, Z.data_ptr(), r, r, Y.data_ptr(), r, s.cuda_stream)


apass()
torch.cuda.synchronize()
# correctness on a column sample
cols = torch.randint(0, n, (4096,), device=dev)
ref = A[:, cols].double().T @ Z
err = float((Y[cols] - ref).abs().max() / ref.abs().max())
evs = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
with ClockSampler(0) as clk:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    evs[0].record(s)
    for i in range(reps):
        apass()
        evs[i + 1].record(s)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
d = [evs[i].elapsed_time(evs[i + 1]) for i in range(reps)]
bytes_ = A.numel() * A.element_size() + (m + n) * r * 8
import os
print(json.dumps({"variant": "fma" if os.environ.get("SPB_K2_FMA") else "dmma", "r": r, "m": m, "n": n,
                  "dtype": str(dt), "relerr": err, "first5_ms": d[:5], "median_ms": statistics.median(d),
                  "last10_ms": statistics.median(d[-10:]), "min_ms": min(d),
                  "GBps_median": bytes_ / statistics.median(d) / 1e6, "GBps_last10": bytes_ / statistics.median(d[-10:]) / 1e6,
                  "wall_s": wall, "clocks": clk.summary()}))

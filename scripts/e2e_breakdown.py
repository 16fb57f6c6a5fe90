"""GPU probe: per-call wall time of the host-buffer power_svd and the share of
the result copies (to_host_many), call by call.  python scripts/e2e_breakdown.py [cfg]"""
import sys
import time
import warnings
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2105_01271_b200 as sp  # noqa: E402
from paper_2105_01271_b200 import device as dv  # noqa: E402
from paper_2105_01271_b200.datagen import CONFIGS, generate_device  # noqa: E402

warnings.simplefilter("ignore")
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
A = generate_device(cfg, torch.device("cuda", 0))
op, cols = sp.grid_injection(cfg.grid, cfg.stride)
pc = sp.PowerConfig(q=cfg.q, columns=cols)
host = np.empty(tuple(A.shape), dtype=np.float64 if A.dtype == torch.float64 else np.float32)
ht = torch.from_numpy(host)
rc = torch.cuda.cudart().cudaHostRegister(ht.data_ptr(), ht.numel() * ht.element_size(), 0)
ht.copy_(A)
torch.cuda.synchronize()
del A
torch.cuda.empty_cache()
orig = dv.to_host_many
spent = {}


def timed(*xs):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = orig(*xs)
    spent["d2h"] = time.perf_counter() - t0
    spent["bytes"] = sum(o.nbytes for o in out)
    return out


dv.to_host_many = timed
for i in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = sp.power_svd(sp.ArraySnapshotStream(host), op, cfg.k, pc)
    dt = time.perf_counter() - t0
    print(f"call {i}: {dt * 1e3:9.2f} ms   result copies {spent['d2h'] * 1e3:8.2f} ms for {spent['bytes'] / 1e6:.1f} MB "
          f"({spent['bytes'] / spent['d2h'] / 1e9:.1f} GB/s)", flush=True)

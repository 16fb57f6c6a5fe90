"""GPU probe: where the end-to-end (host buffers) time goes.

    python scripts/e2e_probe.py [cfg2|cfg3|...]
"""
import sys
import time
import warnings
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2105_01271_b200 as sp  # noqa: E402
from paper_2105_01271_b200.datagen import CONFIGS, generate_device  # noqa: E402
from paper_2105_01271_b200.snapshot_io import _is_pinned, stage_stream  # noqa: E402

warnings.simplefilter("ignore")
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = CONFIGS[name]
dev = torch.device("cuda", 0)
A = generate_device(cfg, dev)
nbytes = A.numel() * A.element_size()
op, cols = sp.grid_injection(cfg.grid, cfg.stride)
pc = sp.PowerConfig(q=cfg.q, columns=cols)


def t(label, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    print(f"{label:58s} {dt * 1e3:9.2f} ms  {nbytes / dt / 1e9:7.1f} GB/s of A", flush=True)
    return out


# (a) torch's pinned allocator, (b) a numpy array registered in place (the bench's e2e buffer)
big = nbytes > 40e9   # one host copy only, raw H2D lands in A itself
hp = None
if not big:
    hp = torch.empty(A.shape, dtype=A.dtype, pin_memory=True)
    hp.copy_(A)
hreg = np.empty(tuple(A.shape), dtype=np.float64 if A.dtype == torch.float64 else np.float32)
treg = torch.from_numpy(hreg)
rc = torch.cuda.cudart().cudaHostRegister(treg.data_ptr(), treg.numel() * treg.element_size(), 0)
treg.copy_(A)
torch.cuda.synchronize()
print("registered rc", int(rc), "is_pinned(registered)", _is_pinned(torch, hreg), flush=True)
d = A if big else torch.empty_like(A)
if not big:
    t("raw H2D copy_ torch-pinned", lambda: d.copy_(hp, non_blocking=True))
t("raw H2D copy_ registered numpy", lambda: d.copy_(torch.from_numpy(hreg), non_blocking=True))
del d
if big:
    del A
    torch.cuda.empty_cache()
for label, hv in ((("torch-pinned", hp.numpy()),) if not big else ()) + (("registered", hreg),):
    t(f"stage only 256 [{label}]", lambda: stage_stream(sp.ArraySnapshotStream(hv), 256))
    t(f"power_svd host stream -> device result [{label}]",
      lambda: sp.power_svd(sp.ArraySnapshotStream(hv), op, cfg.k, pc, return_device=True))
    t(f"power_svd host stream -> numpy result [{label}]",
      lambda: sp.power_svd(sp.ArraySnapshotStream(hv), op, cfg.k, pc))
if big:
    sys.exit(0)
r = sp.power_svd(sp.DeviceSnapshotStream(A), op, cfg.k, pc, return_device=True)
t("device-resident power_svd", lambda: sp.power_svd(sp.DeviceSnapshotStream(A), op, cfg.k, pc, return_device=True), reps=10)
t("D2H of U,S,V (pageable .cpu())", lambda: (r.u.cpu(), r.s.cpu(), r.v.cpu()))

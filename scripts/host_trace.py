"""GPU probe: host-side critical path of one cfg2 power_svd call.
Run with SPB_HOST_TRACE=1: prints the C++ host marks of the last call (us
since the first mark, delta) next to the Python API entry / exit."""
import ctypes
import os
import sys
import time
import warnings
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2105_01271_b200 as sp  # noqa: E402
from paper_2105_01271_b200 import _lib  # noqa: E402
from paper_2105_01271_b200.datagen import CONFIGS, generate_device  # noqa: E402

assert os.environ.get("SPB_HOST_TRACE"), "set SPB_HOST_TRACE=1"
warnings.simplefilter("ignore")
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
A = generate_device(cfg, torch.device("cuda", 0))
op, cols = sp.grid_injection(cfg.grid, cfg.stride)
pc = sp.PowerConfig(q=cfg.q, columns=cols)
lib = _lib.load()
lib.sp_host_trace.restype = ctypes.c_char_p
for _ in range(20):
    sp.power_svd(sp.DeviceSnapshotStream(A), op, cfg.k, pc, return_device=True)
torch.cuda.synchronize()
lib.sp_host_trace()
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.monotonic() * 1e6
    sp.power_svd(sp.DeviceSnapshotStream(A), op, cfg.k, pc, return_device=True)
    t1 = time.monotonic() * 1e6
    tr = lib.sp_host_trace().decode()
    torch.cuda.synchronize()
    t2 = time.monotonic() * 1e6
print(f"python call {t1 - t0:.1f} us, until idle {t2 - t0:.1f} us")
print(tr)

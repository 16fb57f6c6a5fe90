"""Per-call time and free HBM of repeated power_id calls on a BASELINE field
(is the call-to-call spread at cfg5 the workspace pool running out of HBM?).
Usage: SPB_HOST_TRACE=1 python scripts/id_mem_probe.py cfg5 [calls]"""
import gc
import sys
import time
import warnings
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2105_01271_b200 as sp  # noqa: E402
from paper_2105_01271_b200 import _lib  # noqa: E402
from paper_2105_01271_b200.datagen import CONFIGS, generate_device  # noqa: E402

warnings.simplefilter("ignore")
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg5"]
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 8
A = generate_device(cfg, torch.device("cuda", 0))
op, cols = sp.grid_injection(cfg.grid, cfg.stride)
pc = sp.PowerConfig(q=cfg.q, columns=cols)
gc.disable()
import ctypes  # noqa: E402
lib = _lib.load()
lib.sp_host_trace.restype = ctypes.c_char_p
for i in range(calls):
    torch.cuda.synchronize()
    free0, total = torch.cuda.mem_get_info()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lib.sp_host_trace()
    l0 = _lib.launch_count()
    t0 = time.perf_counter()
    e0.record()
    f = sp.power_id(sp.DeviceSnapshotStream(A), op, cfg.k, pc, return_device=True)
    e1.record()
    torch.cuda.synchronize()
    wall = 1e3 * (time.perf_counter() - t0)
    free1, _ = torch.cuda.mem_get_info()
    tr = lib.sp_host_trace().decode()
    print(f"call {i}: launches {_lib.launch_count() - l0}, device {e0.elapsed_time(e1):.1f} ms, wall {wall:.1f} ms, free before/after "
          f"{free0 / 2**30:.1f} / {free1 / 2**30:.1f} GiB of {total / 2**30:.1f}", flush=True)
    if '-v' in sys.argv:
        print(tr, flush=True)
    del f

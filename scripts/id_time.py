"""GPU probe: wall / device time of consecutive power_id calls.  python scripts/id_time.py cfg3|cfg5 [calls]"""
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
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 5
A = generate_device(cfg, torch.device("cuda", 0))
torch.cuda.synchronize()
print("torch reserved GB", torch.cuda.memory_reserved() / 1e9, "allocated", torch.cuda.memory_allocated() / 1e9,
      "free/total", [x / 1e9 for x in torch.cuda.mem_get_info()], flush=True)
op, cols = sp.grid_injection(cfg.grid, cfg.stride)
pc = sp.PowerConfig(q=cfg.q, columns=cols)
for i in range(calls):
    torch.cuda.synchronize()
    l0 = _lib.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    f = sp.power_id(sp.DeviceSnapshotStream(A), op, cfg.k, pc, return_device=True)
    e1.record()
    torch.cuda.synchronize()
    print(f"call {i}: wall {1e3 * (time.perf_counter() - t0):8.1f} ms  events {e0.elapsed_time(e1):8.1f} ms  "
          f"launches {_lib.launch_count() - l0}  free GB {torch.cuda.mem_get_info()[0] / 1e9:.1f}", flush=True)
    del f

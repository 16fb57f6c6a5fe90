"""One warm + one measured power_id call on a BASELINE field (device A), for
ncu launch lists (the summary keeps the second call's launches).
Usage: python scripts/id_call.py cfg3|cfg5"""
import sys
import warnings
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2105_01271_b200 as sp  # noqa: E402
from paper_2105_01271_b200 import _lib  # noqa: E402
from paper_2105_01271_b200.datagen import CONFIGS, generate_device  # noqa: E402

warnings.simplefilter("ignore")
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
A = generate_device(cfg, torch.device("cuda", 0))
op, cols = sp.grid_injection(cfg.grid, cfg.stride)
pc = sp.PowerConfig(q=cfg.q, columns=cols)
for i in range(2):
    l0 = _lib.launch_count()
    f = sp.power_id(sp.DeviceSnapshotStream(A), op, cfg.k, pc, return_device=True)
    torch.cuda.synchronize()
    print(f"call {i}: library launches {_lib.launch_count() - l0}, lift_r {f.r}, bulk_split {f.lifting.bulk_split}",
          flush=True)
    del f

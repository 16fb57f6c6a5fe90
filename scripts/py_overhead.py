"""GPU probe: where the Python mirror spends host time around one power_svd
call (cProfile of warmed calls; argv[1] = BASELINE config)."""
import cProfile
import pstats
import sys
import warnings
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2105_01271_b200 as sp  # noqa: E402
from paper_2105_01271_b200.datagen import CONFIGS, generate_device  # noqa: E402

warnings.simplefilter("ignore")
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
A = generate_device(cfg)
op, cols = sp.grid_injection(cfg.grid, cfg.stride)
pc = sp.PowerConfig(q=cfg.q, columns=cols)


def api():
    return sp.power_svd(sp.DeviceSnapshotStream(A), op, cfg.k, pc, return_device=True)


for _ in range(3):
    api()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    api()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)

"""GPU probe: power_id at a BASELINE config (default cfg3), CUDA-event timed;
PROBE_STEPS=1 brackets one call with cudaProfilerStart/Stop for ncu launch lists."""
import os
import sys
import time
import warnings
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2105_01271_b200 as sp  # noqa: E402
from paper_2105_01271_b200.datagen import CONFIGS, generate_device  # noqa: E402

warnings.simplefilter("ignore")
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
cfg = CONFIGS[name]
if os.environ.get("PROBE_NOISELESS"):
    cfg = cfg.scaled(name=name)  # same shape
    object.__setattr__(cfg, "noise_std", 0.0)
t0 = time.perf_counter()
A = generate_device(cfg)
torch.cuda.synchronize()
print("gen s", time.perf_counter() - t0, flush=True)
op, cols = sp.grid_injection(cfg.grid, cfg.stride)
pc = sp.PowerConfig(q=cfg.q, columns=cols)


def run():
    return sp.power_id(sp.DeviceSnapshotStream(A), op, cfg.k, pc, return_device=True)


run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
f = run()
e1.record()
torch.cuda.synchronize()
print(f"{name} power_id ms {e0.elapsed_time(e1):.1f}  r={f.r}", flush=True)
if int(os.environ.get("PROBE_STEPS", "0")):
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    run()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()

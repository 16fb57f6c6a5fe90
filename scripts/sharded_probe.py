"""GPU probe: per-step time of the column-sharded driver (sharded.py) at
world size 1 over NCCL -- the per-rank cost the N>1 bench pays -- beside the
fused single-GPU pipeline on the same cfg2 slab."""
import os
import sys
import time
import warnings
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2105_01271_b200 as sp  # noqa: E402
from paper_2105_01271_b200.datagen import CONFIGS, coarse_grid_indices, generate_device  # noqa: E402
from paper_2105_01271_b200.sharded import DeviceOps, TorchComm, sharded_power_svd  # noqa: E402

warnings.simplefilter("ignore")
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1)
torch.cuda.set_device(0)
cfg = CONFIGS["cfg2"]
A = generate_device(cfg)
cols = coarse_grid_indices(cfg.grid, cfg.stride)
comm, ops = TorchComm(), DeviceOps()
op, _ = sp.grid_injection(cfg.grid, cfg.stride)
pc = sp.PowerConfig(q=cfg.q, columns=cols)


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


print("sharded world=1 ms", timeit(lambda: sharded_power_svd(A, 0, cols, cfg.k, cfg.q, comm, ops)))
print("fused ms", timeit(lambda: sp.power_svd(sp.DeviceSnapshotStream(A), op, cfg.k, pc, return_device=True)))
u, s, v, r, _ = sharded_power_svd(A, 0, cols, cfg.k, cfg.q, comm, ops)
ref = sp.power_svd(sp.DeviceSnapshotStream(A), op, cfg.k, pc, return_device=True)
print("kept", r, "max |ds|/s1", float((torch.as_tensor(s, device="cuda") - ref.s).abs().max() / ref.s[0]))
if os.environ.get("PROBE_CPROFILE"):
    import cProfile
    import pstats
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(10):
        sharded_power_svd(A, 0, cols, cfg.k, cfg.q, comm, ops)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)
if int(os.environ.get("PROBE_STEPS", "0")):
    torch.cuda.cudart().cudaProfilerStart()
    sharded_power_svd(A, 0, cols, cfg.k, cfg.q, comm, ops)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
dist.destroy_process_group()

"""GPU probe: does the cfg2 per-call time depend on what ran before it in the
process (allocator state, a cfg4-sized call, the e2e leg's page-locking)?"""
import gc
import sys
import time
import warnings
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2105_01271_b200 as sp  # noqa: E402
from paper_2105_01271_b200 import _lib  # noqa: E402
from paper_2105_01271_b200.datagen import CONFIGS, generate_device  # noqa: E402

warnings.simplefilter("ignore")
dev = torch.device("cuda", 0)


def loop(label, cfgname="cfg2", reps=20):
    cfg = CONFIGS[cfgname]
    A = generate_device(cfg, dev)
    op, cols = sp.grid_injection(cfg.grid, cfg.stride)
    pc = sp.PowerConfig(q=cfg.q, columns=cols)

    def f():
        return sp.power_svd(sp.DeviceSnapshotStream(A), op, cfg.k, pc, return_device=True)
    t0 = time.perf_counter()
    n = 0
    while n < 3 or time.perf_counter() - t0 < 0.3:
        r = f()
        n += 1
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = _lib.launch_count()
    w0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        r = f()
    e1.record()
    torch.cuda.synchronize()
    w = (time.perf_counter() - w0) / reps * 1e3
    print(f"{label:50s} {cfgname} events {e0.elapsed_time(e1) / reps:7.3f} ms  wall {w:7.3f} ms  "
          f"launches/call {(_lib.launch_count() - l0) / reps:.1f}  gc={gc.isenabled()}", flush=True)
    del r, A


loop("fresh")
gc.disable()
loop("fresh, gc disabled")
gc.enable()
x = torch.empty(int(100e9), dtype=torch.uint8, device=dev)
x.zero_()
del x
torch.cuda.empty_cache()
loop("after a 100 GB torch tensor came and went")
loop("cfg4 call", "cfg4", reps=3)
gc.collect()
torch.cuda.empty_cache()
loop("after cfg4")
from bench import ClockSampler  # noqa: E402
with ClockSampler(0) as clk:
    loop("inside a ClockSampler region")
print(clk.summary())
loop("after the ClockSampler region")
cfg = CONFIGS["cfg2"]
A = generate_device(cfg, dev)
op, cols = sp.grid_injection(cfg.grid, cfg.stride)
pc = sp.PowerConfig(q=cfg.q, columns=cols)
host = np.empty((cfg.m, cfg.n))
ht = torch.from_numpy(host)
rc = torch.cuda.cudart().cudaHostRegister(ht.data_ptr(), ht.numel() * 8, 0)
ht.copy_(A)
torch.cuda.synchronize()
for i in range(4):
    t0 = time.perf_counter()
    out = sp.power_svd(sp.ArraySnapshotStream(host), op, cfg.k, pc)
    print(f"e2e call {i}: {(time.perf_counter() - t0) * 1e3:.2f} ms", flush=True)
del out
loop("after e2e calls (host still registered)")
torch.cuda.cudart().cudaHostUnregister(ht.data_ptr())
loop("after unregistering")

import time, torch, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_01271_b200.device import to_host_many
v = torch.randn(65536, 50, dtype=torch.float64, device="cuda"); u = torch.randn(2000, 50, dtype=torch.float64, device="cuda")
for i in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter(); a, b = to_host_many(u, v); print("to_host_many ms", (time.perf_counter() - t0) * 1e3)
    del a, b
h = torch.empty(v.shape, dtype=v.dtype, pin_memory=True)
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); h.copy_(v, non_blocking=True); torch.cuda.synchronize(); print("reused pinned ms", (time.perf_counter() - t0) * 1e3)
import numpy as np
for i in range(3):
    t0 = time.perf_counter(); x = np.array(h.numpy(), copy=True); print("host memcpy 26MB ms", (time.perf_counter() - t0) * 1e3)
for i in range(3):
    t0 = time.perf_counter(); hh = torch.empty(v.shape, dtype=v.dtype, pin_memory=True); print("pinned alloc ms", (time.perf_counter() - t0) * 1e3); del hh

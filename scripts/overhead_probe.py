"""GPU probe: host overhead of the Python mirror vs the bare C pipeline call (default cfg2;
argv[1] names another BASELINE config).  PROBE_STEPS=n brackets n API calls with
cudaProfilerStart/Stop for ncu launch lists."""
import sys, time, warnings
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2105_01271_b200 as sp
from paper_2105_01271_b200 import _lib
from paper_2105_01271_b200.datagen import CONFIGS
from paper_2105_01271_b200.datagen import generate_device
warnings.simplefilter("ignore")
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]; dev = torch.device("cuda", 0)
A = generate_device(cfg, dev)
op, cols = sp.grid_injection(cfg.grid, cfg.stride)
TAG = 0 if A.dtype == torch.float64 else 1
pc = sp.PowerConfig(q=1, columns=cols)
def api():
    return sp.power_svd(sp.DeviceSnapshotStream(A), op, cfg.k, pc, return_device=True)
for _ in range(3): api()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10): api()
torch.cuda.synchronize()
print("api wall ms", (time.perf_counter() - t0) / 10 * 1e3)
# bare C call with pre-gathered C
idx, w, depth, om = op.device_tables()
dcols = torch.from_numpy(cols).to(dev)
C = torch.empty((cfg.m, cols.size), dtype=torch.float64, device=dev)
s = torch.cuda.current_stream().cuda_stream
_lib.call("sp_apply_stencil", A.data_ptr(), TAG, cfg.m, cfg.n, cfg.n, dcols.data_ptr(), None, 1, cols.size, 1, C.data_ptr(), cols.size, s)
U = torch.empty((cfg.m, cfg.k), dtype=torch.float64, device=dev); S = torch.empty(cfg.k, dtype=torch.float64, device=dev); V = torch.empty((cfg.n, cfg.k), dtype=torch.float64, device=dev)
info = _lib.new_info()
def bare():
    _lib.call("sp_power_svd", A.data_ptr(), TAG, cfg.m, cfg.n, cfg.n, idx.data_ptr(), w.data_ptr(), depth, op.n_c, None, 0,
              dcols.data_ptr(), cols.size, 1, cfg.k, C.data_ptr(), C.data_ptr(), 3, U.data_ptr(), S.data_ptr(), V.data_ptr(), _lib.info_ptr(info), s)
for _ in range(3): bare()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10): bare()
torch.cuda.synchronize()
print("bare C wall ms", (time.perf_counter() - t0) / 10 * 1e3, "launches", info[_lib.INFO_LAUNCHES])
# step-only section for ncu launch lists: PROBE_STEPS API calls, nothing else
import os
n = int(os.environ.get("PROBE_STEPS", "0"))
if n:
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    for _ in range(n): api()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()

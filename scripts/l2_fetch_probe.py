"""GPU probe: cudaLimitMaxL2FetchGranularity (32 / 64 / 128 B) against the
stride-8 coarse-grid gather of cfg4 (one grid point per 64 bytes) and the A pass."""
import ctypes
import subprocess
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
torch.zeros(1, device="cuda")
rt = ctypes.CDLL("libcudart.so.12")
val = ctypes.c_size_t(0)
rt.cudaDeviceGetLimit(ctypes.byref(val), 5)
print("default cudaLimitMaxL2FetchGranularity:", val.value, flush=True)
for g in (int(a) for a in sys.argv[1:] or ["64", "32", "128"]):
    rc = rt.cudaDeviceSetLimit(5, ctypes.c_size_t(g))
    rt.cudaDeviceGetLimit(ctypes.byref(val), 5)
    print(f"--- set {g}: rc {rc}, now {val.value}", flush=True)
    sys.argv = ["gather_probe.py", "cfg4", "cfg2"]
    exec(open(Path(__file__).resolve().parent / "gather_probe.py").read())
    from paper_2105_01271_b200 import _lib
    m, n, r = 2000, 1 << 20, 8
    A = torch.randn(m, n, dtype=torch.float64, device="cuda")
    Z = torch.randn(m, r, dtype=torch.float64, device="cuda")
    Y = torch.empty(n, r, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()
    f = lambda: _lib.call("sp_skinny_atz", A.data_ptr(), _lib.SP_F64, m, n, n, Z.data_ptr(), r, r, Y.data_ptr(), r, st.cuda_stream)
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    torch.cuda.synchronize()
    print(f"K2 {m}x{n}: {e0.elapsed_time(e1) / 10:.3f} ms  {m * n * 8 / e0.elapsed_time(e1) * 10 / 1e6:.0f} GB/s", flush=True)
    del A, Z, Y

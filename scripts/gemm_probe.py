"""GPU probe: the library's FP64 DMMA GEMM (sp_gemm) against cuBLAS DGEMM
(torch.matmul, float64) at the sketch-side product shapes of cfg2..cfg5, plus
a square DGEMM for the FP64 tensor peak.  Warmed CUDA-event timings."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_01271_b200 import _lib  # noqa: E402

dev = torch.device("cuda", 0)
st = torch.cuda.current_stream()
s = st.cuda_stream
P = lambda t: t.data_ptr()  # noqa: E731


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


n = 8192
a = torch.randn(n, n, dtype=torch.float64, device=dev)
b = torch.randn(n, n, dtype=torch.float64, device=dev)
us = timeit(lambda: a @ b, 3)
print(f"cuBLAS DGEMM {n}^3: {us:9.1f} us  {2 * n**3 / us / 1e6:6.1f} TF/s", flush=True)
c = torch.empty_like(a)
us = timeit(lambda: _lib.call("sp_gemm", 0, 0, n, n, n, 1.0, P(a), n, P(b), n, 0.0, P(c), n, s), 3)
print(f"sp_gemm DGEMM {n}^3: {us:9.1f} us  {2 * n**3 / us / 1e6:6.1f} TF/s", flush=True)
del a, b, c
for name, m, nc in (("cfg2", 2000, 4096), ("cfg3", 5000, 4096), ("cfg4", 10000, 16384), ("cfg5", 2000, 262144)):
    C = torch.randn(m, nc, dtype=torch.float64, device=dev)
    Q = torch.randn(m, 32, dtype=torch.float64, device=dev)
    Pm = torch.randn(nc, 32, dtype=torch.float64, device=dev)
    Z = torch.empty(nc, 32, dtype=torch.float64, device=dev)
    Y = torch.empty(m, 32, dtype=torch.float64, device=dev)
    fl = 2 * m * nc * 32
    t1 = timeit(lambda: _lib.call("sp_gemm", 1, 0, nc, 32, m, 1.0, P(C), nc, P(Q), 32, 0.0, P(Z), 32, s))
    t2 = timeit(lambda: torch.matmul(C.t(), Q, out=Z))
    t3 = timeit(lambda: _lib.call("sp_gemm", 0, 0, m, 32, nc, 1.0, P(C), nc, P(Pm), 32, 0.0, P(Y), 32, s))
    t4 = timeit(lambda: torch.matmul(C, Pm, out=Y))
    gb = m * nc * 8 / 1e3
    print(f"{name} Z=C^T Q: sp {t1:8.1f} us ({fl / t1 / 1e6:5.1f} TF/s, {gb / t1:5.0f} GB/s)  cuBLAS {t2:8.1f} us"
          f" | Y=C P: sp {t3:8.1f} us ({fl / t3 / 1e6:5.1f} TF/s)  cuBLAS {t4:8.1f} us", flush=True)
    del C, Q, Pm, Z, Y
    torch.cuda.empty_cache()

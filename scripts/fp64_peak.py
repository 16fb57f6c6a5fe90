"""FP64 roofline denominators for the ID's compute-bound kernels: the library's
DMMA GEMM (sp_gemm) and cuBLAS DGEMM at 8192^3, the nearly-exact product
(sp_gemm_exact, two DMMA levels) at the cfg3 enrichment shape, warmed CUDA
events.  Prints one JSON line."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_01271_b200 import _lib  # noqa: E402

dev = torch.device("cuda", 0)
st = torch.cuda.current_stream()
s = st.cuda_stream
P = lambda t: t.data_ptr()  # noqa: E731


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


out = {}
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device=dev)
b = torch.randn(n, n, dtype=torch.float64, device=dev)
c = torch.empty_like(a)
out["cublas_dgemm_8192_tflops"] = 2 * n ** 3 / timeit(lambda: torch.matmul(a, b, out=c)) / 1e12
out["sp_gemm_dmma_8192_tflops"] = 2 * n ** 3 / timeit(
    lambda: _lib.call("sp_gemm", 0, 0, n, n, n, 1.0, P(a), n, P(b), n, 0.0, P(c), n, s)) / 1e12
del a, b, c
m, nc = 5000, 4096
C = torch.randn(m, nc, dtype=torch.float64, device=dev)
T = torch.randn(nc, nc, dtype=torch.float64, device=dev)
hi = torch.empty(m, nc, dtype=torch.float64, device=dev)
lo = torch.empty_like(hi)
fl = 2 * m * nc * nc
t_plain = timeit(lambda: _lib.call("sp_gemm", 0, 0, m, nc, nc, 1.0, P(C), nc, P(T), nc, 0.0, P(hi), nc, s))
t_exact = timeit(lambda: _lib.call("sp_gemm_exact", 0, m, nc, nc, P(C), nc, P(T), None, nc, P(hi), P(lo), nc, s))
out.update(cfg3_enrichment_plain_ms=t_plain * 1e3, cfg3_enrichment_exact_ms=t_exact * 1e3,
           cfg3_enrichment_plain_tflops=fl / t_plain / 1e12,
           exact_over_plain=t_exact / t_plain,
           note="sp_gemm_exact = exact head level (depth K) + FP64 rest (depth 2K) on DMMA, 3x the plain "
                "GEMM's flops; DMMA (mma.sync.m8n8k4.f64) is the only FP64 tensor path on sm_100a (tcgen05 has no f64 kind)")
print(json.dumps(out))

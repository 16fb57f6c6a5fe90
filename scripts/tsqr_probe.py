"""GPU probe: time the sketch-side building blocks in isolation (CUDA events,
warm): TSQR of 2000x32 / 4096x32 / 65536x7, Jacobi 32x32 / 7x7.  Build with
SPB_NVCC_EXTRA=-DSPB_TSQR_TRACE for per-step cycle counts of the TSQR leaf."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_01271_b200 import _lib  # noqa: E402

dev = torch.device("cuda", 0)
s = torch.cuda.current_stream()
g = torch.Generator(device=dev).manual_seed(0)


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
    return e0.elapsed_time(e1) / n * 1e3


once = "--once" in sys.argv
for rows, cols in [(2000, 32), (4096, 32), (65536, 7)]:
    x = torch.randn(rows, cols, dtype=torch.float64, device=dev, generator=g)
    q = torch.empty_like(x)
    r = torch.empty(cols, cols, dtype=torch.float64, device=dev)
    fn = lambda: _lib.call("sp_tsqr", rows, cols, x.data_ptr(), cols, q.data_ptr(), cols, r.data_ptr(), cols,
                           s.cuda_stream)
    if once:
        fn(); torch.cuda.synchronize(); continue
    print(f"tsqr {rows}x{cols}: {timeit(fn):.1f} us")
for n in [32, 7]:
    m = torch.randn(n, n, dtype=torch.float64, device=dev, generator=g)
    u = torch.empty_like(m); v = torch.empty_like(m); sv = torch.empty(n, dtype=torch.float64, device=dev)
    fn = lambda: _lib.call("sp_jacobi_svd", n, m.data_ptr(), n, u.data_ptr(), n, sv.data_ptr(), v.data_ptr(), n,
                           s.cuda_stream)
    if not once:
        print(f"jacobi {n}x{n}: {timeit(fn):.1f} us")

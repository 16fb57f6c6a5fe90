"""GPU probe: warmed CUDA-event timings of the C-ABI primitives at the cfg2
pipeline shapes (what each step of power_svd spends its time on)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_01271_b200 import _lib  # noqa: E402

dev = torch.device("cuda", 0)
st = torch.cuda.current_stream()
s = st.cuda_stream
g = torch.Generator(device=dev).manual_seed(0)


def rnd(*shape):
    return torch.randn(*shape, dtype=torch.float64, device=dev, generator=g)


def graded(rows, cols, decay=1e-1):
    """rows x cols with singular values decaying geometrically (rank deficient)."""
    U, _ = torch.linalg.qr(rnd(rows, cols))
    V, _ = torch.linalg.qr(rnd(cols, cols))
    sv = decay ** torch.arange(cols, dtype=torch.float64, device=dev)
    return (U * sv) @ V.T


def timeit(name, fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0 = _lib.launch_count()
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    nl = (_lib.launch_count() - n0) / reps
    print(f"{name:52s} {e0.elapsed_time(e1) / reps * 1e3:9.1f} us  {nl:5.1f} launches", flush=True)


P = lambda t: t.data_ptr()  # noqa: E731
m, nc, b, n, r = 2000, 4096, 32, 65536, 7
C = rnd(m, nc)
Om = rnd(nc, b)
Y = rnd(m, b)
Q = rnd(m, b)
Z = rnd(nc, b)
G = rnd(64, 64)
timeit("gemm Y=C Om (2000x4096 @ 4096x32)",
       lambda: _lib.call("sp_gemm", 0, 0, m, b, nc, 1.0, P(C), nc, P(Om), b, 0.0, P(Y), b, s))
timeit("gemm Z=C^T Q (4096x2000 @ 2000x32)",
       lambda: _lib.call("sp_gemm", 1, 0, nc, b, m, 1.0, P(C), nc, P(Q), b, 0.0, P(Z), b, s))
for rows, cols in ((2000, 32), (4096, 32), (n, r), (n, 32)):
    X = graded(rows, cols)
    Qo = torch.empty_like(X)
    R = torch.empty((cols, cols), dtype=torch.float64, device=dev)
    timeit(f"tsqr {rows}x{cols}",
           lambda: _lib.call("sp_tsqr", rows, cols, P(X), cols, P(Qo), cols, P(R), cols, s))
    Xw = rnd(rows, cols)
    timeit(f"qr_tall well-conditioned (cholqr2) {rows}x{cols}",
           lambda: _lib.call("sp_qr_tall", rows, cols, P(Xw), cols, P(Qo), cols, P(R), cols, 1, s))
for rows, c, d in ((n, 7, 7), (4096, 32, 32), (n, 32, 32), (n, 64, 64)):
    X = rnd(rows, c)
    Yv = rnd(rows, d)
    timeit(f"gram X^T Y {rows}x{c} {rows}x{d}",
           lambda: _lib.call("sp_gemm", 1, 0, c, d, rows, 1.0, P(X), c, P(Yv), d, 0.0, P(G), 64, s))
for rows, c, d in ((n, 7, 7), (n, 7, 43), (4096, 32, 32), (n, 32, 32), (n, 64, 64)):
    X = rnd(rows, c)
    M = rnd(c, d)
    O = rnd(rows, d)
    timeit(f"mul X M {rows}x{c} @ {c}x{d}",
           lambda: _lib.call("sp_gemm", 0, 0, rows, d, c, 1.0, P(X), c, P(M), d, 0.0, P(O), d, s))
for k in (7, 16, 32, 64):
    M = graded(k, k, 0.3)
    U = torch.empty_like(M)
    V = torch.empty_like(M)
    S = torch.empty(k, dtype=torch.float64, device=dev)
    timeit(f"jacobi_svd {k}x{k}",
           lambda: _lib.call("sp_jacobi_svd", k, P(M), k, P(U), k, P(S), P(V), k, s))
A = rnd(m, n)
Zr = rnd(m, r)
Yr = torch.empty((n, r), dtype=torch.float64, device=dev)
timeit("skinny_atz A^T Z (2000x65536, r=7)",
       lambda: _lib.call("sp_skinny_atz", P(A), 0, m, n, n, P(Zr), r, r, P(Yr), r, s))
cols = torch.arange(0, n, 16, dtype=torch.int64, device=dev)
Cg = torch.empty((m, cols.numel()), dtype=torch.float64, device=dev)
timeit("apply_stencil gather 2000 x 4096",
       lambda: _lib.call("sp_apply_stencil", P(A), 0, m, n, n, P(cols), None, 1, cols.numel(), 1, P(Cg),
                         cols.numel(), s))

"""GPU probe: the coarse-column gather (K1) and the fused gather + SRHT test
block at the BASELINE grid shapes (cfg2: 256^2 stride 4; cfg4: 1024^2 stride 8,
first M rows; cfg5: 256^3 stride 4 f32, first M rows).  Warmed CUDA-event
timings and the sector-rate GB/s of the gather."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_01271_b200 import _lib  # noqa: E402
from paper_2105_01271_b200.datagen import coarse_grid_indices  # noqa: E402

dev = torch.device("cuda", 0)
st = torch.cuda.current_stream()
s = st.cuda_stream
P = lambda t: t.data_ptr()  # noqa: E731


def timeit(name, fn, nbytes, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    print(f"{name:60s} {us:9.1f} us  {nbytes / us / 1e3:7.0f} GB/s(sector)", flush=True)


which = sys.argv[1:] or ["cfg2", "cfg4", "cfg5"]
for name, grid, stride, m, dt in (("cfg2", (256, 256), 4, 2000, torch.float64),
                                  ("cfg4", (1024, 1024), 8, 2000, torch.float64),
                                  ("cfg5", (256, 256, 256), 4, 1000, torch.float32)):
    if name not in which:
        continue
    cols = torch.from_numpy(coarse_grid_indices(grid, stride)).to(dev)
    n = 1
    for g in grid:
        n *= g
    nc = cols.numel()
    A = torch.randn(m, n, dtype=dt, device=dev)
    tag = 1 if dt == torch.float64 else 0
    tag = _lib.SP_F64 if dt == torch.float64 else _lib.SP_F32
    esz = A.element_size()
    sec = max(1, 32 // (stride * esz))  # grid points per 32-B sector along x
    nbytes = m * (nc // sec) * 32
    C = torch.empty(m, nc, dtype=torch.float64, device=dev)
    Y = torch.empty(m, 32, dtype=torch.float64, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    w = torch.ones(nc, dtype=torch.float64, device=dev)
    timeit(f"{name} K1 gather {m}x{nc}", lambda: _lib.call(
        "sp_apply_stencil", P(A), tag, m, n, n, P(cols), P(w), 1, nc, 1, P(C), nc, s), nbytes)
    if nc <= 16384:
        timeit(f"{name} gather+SRHT {m}x{nc}", lambda: _lib.call(
            "sp_srht_gather", P(A), tag, m, n, P(cols), nc, P(C), nc, 32, 7, P(Y), 32, P(flag), s), nbytes)
        timeit(f"{name} SRHT of C {m}x{nc}", lambda: _lib.call(
            "sp_srht_sketch", m, nc, P(C), nc, 32, 7, P(Y), 32, P(flag), s), m * nc * 8)
    del A
    torch.cuda.empty_cache()

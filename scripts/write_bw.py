"""GPU probe: HBM write-only and read-only bandwidth (torch fill_ / sum) vs copy,
to set the bound of the output passes (finish_rows writes U and V)."""
import torch

dev = torch.device("cuda", 0)
st = torch.cuda.current_stream()


def t(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps / 1e3


for gb in (1.68, 13.4):
    n = int(gb * 1e9 / 8)
    x = torch.empty(n, dtype=torch.float64, device=dev)
    y = torch.empty(n, dtype=torch.float64, device=dev)
    s = t(lambda: x.fill_(1.0))
    print(f"{gb} GB fill (write only): {gb / s:7.0f} GB/s", flush=True)
    s = t(lambda: x.sum())
    print(f"{gb} GB sum (read only):   {gb / s:7.0f} GB/s", flush=True)
    s = t(lambda: y.copy_(x))
    print(f"{gb} GB copy (r+w):        {2 * gb / s:7.0f} GB/s", flush=True)
    del x, y
    torch.cuda.empty_cache()

"""GPU probe: host->device bandwidth of the staging paths."""
import time, torch, numpy as np
n = 1 << 27  # 1 GiB of f64
h = torch.empty(n, dtype=torch.float64, pin_memory=True); h.fill_(1.0)
d = torch.empty(n, dtype=torch.float64, device="cuda")
def bw(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return n * 8 * reps / (time.perf_counter() - t0) / 1e9
print("pinned tensor copy_        GB/s", bw(lambda: d.copy_(h, non_blocking=True)))
hv = h.numpy()
print("from_numpy(pinned) copy_   GB/s", bw(lambda: d.copy_(torch.from_numpy(hv), non_blocking=True)))
blk = 256 * 65536
def chunks():
    for o in range(0, n, blk):
        d[o:o + blk].copy_(torch.from_numpy(hv[o:o + blk]), non_blocking=True)
print("from_numpy chunks 134MB    GB/s", bw(chunks))
hp = np.ones(n)  # pageable
print("pageable numpy copy_       GB/s", bw(lambda: d.copy_(torch.from_numpy(hp), non_blocking=True), reps=2))
print("is_pinned(from_numpy(pinned view))", torch.from_numpy(hv[:10]).is_pinned())

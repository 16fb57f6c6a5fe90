"""GPU-box probe: host->device ingest options for a pageable numpy array --
threaded memcpy into pinned buffers (numpy copyto / ctypes memmove), and
page-locking the caller's chunk in place (cudaHostRegister) then DMA."""
import ctypes, time, json
from concurrent.futures import ThreadPoolExecutor
import numpy as np, torch
cr = torch.cuda.cudart()
src = np.random.default_rng(0).standard_normal((2000, 65536))   # 1 GB pageable
pool = ThreadPoolExecutor(16)
out = {}
def split(n, parts):
    return [(n * i // parts, n * (i + 1) // parts) for i in range(parts)]
dst = torch.empty(64 << 20, dtype=torch.uint8, pin_memory=True)
dp = dst.data_ptr()
for nt in (1, 4, 8, 16):
    t0 = time.perf_counter()
    for c0 in range(0, 2000, 128):
        sub = src[c0:c0 + 128]
        nb = sub.nbytes
        futs = [pool.submit(ctypes.memmove, dp + a, sub.ctypes.data + a, b - a) for a, b in split(nb, nt)]
        for f in futs:
            f.result()
    out[f"memmove_{nt}thr_GBps"] = src.nbytes / (time.perf_counter() - t0) / 1e9
# register in place, whole array
t0 = time.perf_counter()
rc = cr.cudaHostRegister(src.ctypes.data, src.nbytes, 0)
out["register_1GB_s"] = time.perf_counter() - t0
d = torch.empty(src.shape, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
d.copy_(torch.from_numpy(src), non_blocking=True)
torch.cuda.synchronize()
out["h2d_registered_GBps"] = src.nbytes / (time.perf_counter() - t0) / 1e9
t0 = time.perf_counter()
cr.cudaHostUnregister(src.ctypes.data)
out["unregister_1GB_s"] = time.perf_counter() - t0
# chunked register -> DMA -> unregister (64 MB chunks)
t0 = time.perf_counter()
s = torch.cuda.Stream()
for c0 in range(0, 2000, 128):
    sub = src[c0:c0 + 128]
    cr.cudaHostRegister(sub.ctypes.data, sub.nbytes, 0)
    with torch.cuda.stream(s):
        d[c0:c0 + 128].copy_(torch.from_numpy(sub), non_blocking=True)
    s.synchronize()
    cr.cudaHostUnregister(sub.ctypes.data)
out["chunked_register_dma_GBps"] = src.nbytes / (time.perf_counter() - t0) / 1e9
print(json.dumps(out))

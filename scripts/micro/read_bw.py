import torch, time
a = torch.randn(2000, 65536, dtype=torch.float64, device="cuda")
b = torch.empty_like(a)
for name, f in [("sum", lambda: a.sum()), ("amax", lambda: a.abs().amax() if False else a.amax()), ("copy", lambda: b.copy_(a))]:
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    nb = a.numel() * 8 * (2 if name == "copy" else 1)
    print(name, f"{ms*1e3:.1f} us", f"{nb/ms/1e6:.0f} GB/s")

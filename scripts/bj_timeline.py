"""GPU probe: kernel-time breakdown (torch.profiler) of thin_svd on a wide
full-rank core (the block-Jacobi path).  Usage: python scripts/bj_timeline.py M N"""
import collections, json, sys, tempfile
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2105_01271_b200 as sp
m, n = int(sys.argv[1]), int(sys.argv[2])
x = torch.from_numpy(np.random.default_rng(0).standard_normal((m, n)) * np.logspace(0, -6, n)[None, :]).cuda()
sp.thin_svd(x[:300, :200].contiguous())
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    sp.thin_svd(x)
    torch.cuda.synchronize()
path = Path(tempfile.mkdtemp()) / "t.json"
prof.export_chrome_trace(str(path))
ev = [e for e in json.loads(path.read_text())["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
span = ev[-1]["ts"] + ev[-1]["dur"] - ev[0]["ts"]
agg = collections.defaultdict(lambda: [0, 0.0])
for e in ev:
    k = e["name"].replace("(anonymous namespace)::", "").split("(")[0][:70]
    agg[k][0] += 1
    agg[k][1] += e["dur"]
print(f"thin_svd {m}x{n}: span {span / 1e3:.1f} ms, {len(ev)} kernels")
for k, (c, d) in sorted(agg.items(), key=lambda x: -x[1][1])[:15]:
    print(f"{d / 1e3:9.2f} ms {c:6d} {d / max(c, 1):9.1f} us/launch  {k}")

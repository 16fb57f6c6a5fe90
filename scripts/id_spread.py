"""GPU probe: where does the call-to-call spread of power_id come from?  Profiles
several calls (CUPTI via torch.profiler), one trace each, and prints per call the
device span, the sum of kernel times, the idle time and the kernels whose total
moved most against the fastest call.  Usage: python scripts/id_spread.py [cfg5] [calls]"""
import collections
import json
import sys
import tempfile
import warnings
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2105_01271_b200 as sp  # noqa: E402
from paper_2105_01271_b200.datagen import CONFIGS, generate_device  # noqa: E402

warnings.simplefilter("ignore")
name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 6
cfg = CONFIGS[name]
A = generate_device(cfg, torch.device("cuda", 0))
op, cols = sp.grid_injection(cfg.grid, cfg.stride)
pc = sp.PowerConfig(q=cfg.q, columns=cols)


def api():
    return sp.power_id(sp.DeviceSnapshotStream(A), op, cfg.k, pc, return_device=True)


for _ in range(3):
    api()
torch.cuda.synchronize()
recs = []
for i in range(calls):
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        api()
        torch.cuda.synchronize()
    path = Path(tempfile.mkdtemp()) / "trace.json"
    prof.export_chrome_trace(str(path))
    ev = json.loads(path.read_text())["traceEvents"]
    kern = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
    span = kern[-1]["ts"] + kern[-1]["dur"] - kern[0]["ts"]
    busy, end = 0.0, kern[0]["ts"]
    gaps = []
    for e in kern:
        if e["ts"] > end:
            gaps.append((e["ts"] - end, e["name"].split("(")[0][-40:]))
        lo = max(e["ts"], end)
        hi = e["ts"] + e["dur"]
        if hi > lo:
            busy += hi - lo
            end = hi
    agg = collections.defaultdict(lambda: [0, 0.0])
    for e in kern:
        k = e["name"].replace("(anonymous namespace)::", "").split("(")[0][:60]
        agg[k][0] += 1
        agg[k][1] += e["dur"]
    gaps.sort(reverse=True)
    recs.append((span, busy, agg, gaps[:5], len(kern)))
    print(f"call {i}: span {span / 1e3:.1f} ms, busy {busy / 1e3:.1f} ms, idle {(span - busy) / 1e3:.1f} ms, "
          f"{len(kern)} launches; largest gaps (us, before): {[(round(g), n) for g, n in gaps[:5]]}", flush=True)
best = min(recs, key=lambda r: r[0])
for i, (span, busy, agg, _, _) in enumerate(recs):
    diff = sorted(((agg[k][1] - best[2].get(k, [0, 0.0])[1], k) for k in agg), reverse=True)[:4]
    print(f"call {i}: +{(span - best[0]) / 1e3:.1f} ms vs fastest; kernels: " +
          ", ".join(f"{k} +{d / 1e3:.1f} ms" for d, k in diff))

"""GPU probe: kernel-time breakdown of one power_id call (CUPTI via
torch.profiler), aggregated by kernel name.  Usage: python scripts/id_timeline.py [cfg3|cfg5]"""
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
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
cfg = CONFIGS[name]
A = generate_device(cfg, torch.device("cuda", 0))
op, cols = sp.grid_injection(cfg.grid, cfg.stride)
pc = sp.PowerConfig(q=cfg.q, columns=cols)


def api():
    return sp.power_id(sp.DeviceSnapshotStream(A), op, cfg.k, pc, return_device=True)


api()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    api()
    torch.cuda.synchronize()
path = Path(tempfile.mkdtemp()) / "trace.json"
prof.export_chrome_trace(str(path))
ev = json.loads(path.read_text())["traceEvents"]
kern = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
span = kern[-1]["ts"] + kern[-1]["dur"] - kern[0]["ts"]
agg = collections.defaultdict(lambda: [0, 0.0])
for e in kern:
    k = e["name"].replace("(anonymous namespace)::", "").split("(")[0][:80]
    agg[k][0] += 1
    agg[k][1] += e["dur"]
print(f"{name} power_id: device span {span / 1e3:.1f} ms, {len(kern)} launches")
for k, (c, d) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{d / 1e3:9.2f} ms {c:6d}  {k}")

"""GPU probe: warm timeline of one power_svd call (CUPTI via torch.profiler).

Unlike the ncu launch list (cold cache, serialised), this shows the kernels as
they run inside the pipeline, with the idle gaps between them (host syncs,
launch latency).  Usage: python scripts/timeline.py [cfg2] [calls]
Prints, for the last profiled call, each kernel's start offset, duration and
the gap before it, then totals."""
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
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = CONFIGS[name]
dev = torch.device("cuda", 0)
A = generate_device(cfg, dev)
op, cols = sp.grid_injection(cfg.grid, cfg.stride)
pc = sp.PowerConfig(q=cfg.q, columns=cols)


def api():
    return sp.power_svd(sp.DeviceSnapshotStream(A), op, cfg.k, pc, return_device=True)


for _ in range(5):
    api()
torch.cuda.synchronize()
marks = []
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU,
                                        torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(calls):
        torch.cuda.synchronize()
        with torch.profiler.record_function("CALL"):
            api()
        torch.cuda.synchronize()
path = Path(tempfile.mkdtemp()) / "trace.json"
prof.export_chrome_trace(str(path))
ev = json.loads(path.read_text())["traceEvents"]
kern = sorted([e for e in ev if e.get("cat") == "kernel"], key=lambda e: e["ts"])
memc = [e for e in ev if e.get("cat") in ("gpu_memcpy", "gpu_memset")]
callw = sorted([e for e in ev if e.get("name") == "CALL" and e.get("cat") == "user_annotation"],
               key=lambda e: e["ts"])
last = callw[-1]
t0 = last["ts"]
# the call returns before its last kernels finish (no trailing sync): take
# everything launched after its start (the profiled loop syncs after each call)
ks = [e for e in kern + memc if t0 <= e["ts"]]
ks.sort(key=lambda e: e["ts"])
first = ks[0]["ts"]
prev_end = first
busy = 0.0
print(f"{name}: host call wall {last['dur']:.1f} us; device span {ks[-1]['ts'] + ks[-1]['dur'] - first:.1f} us")
print(f"{'start':>8} {'dur':>7} {'gap':>6}  kernel")
for e in ks:
    gap = e["ts"] - prev_end
    print(f"{e['ts'] - first:8.1f} {e['dur']:7.1f} {gap:6.1f}  {e['name'][:90]}")
    prev_end = max(prev_end, e["ts"] + e["dur"])
    busy += e["dur"]
print(f"busy {busy:.1f} us, span {prev_end - first:.1f} us, idle {prev_end - first - busy:.1f} us, "
      f"{sum(1 for e in ks if e.get('cat') == 'kernel')} kernels")

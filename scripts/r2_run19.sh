timeout 600 python scripts/id_timeline.py cfg3 2>/dev/null | head -22
python - <<'PY'
import sys, json, tempfile, collections, warnings
from pathlib import Path
import torch
sys.path.insert(0, '.')
import __graft_entry__ as g
g.smoke()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    g.smoke()
    torch.cuda.synchronize()
p = Path(tempfile.mkdtemp()) / "t.json"; prof.export_chrome_trace(str(p))
ev = [e for e in json.loads(p.read_text())["traceEvents"] if e.get("cat") == "kernel"]
agg = collections.defaultdict(lambda: [0, 0.0])
for e in ev:
    k = e["name"].replace("(anonymous namespace)::", "").split("(")[0][:60]; agg[k][0] += 1; agg[k][1] += e["dur"]
print("smoke kernels:", len(ev), "total us", sum(e["dur"] for e in ev))
for k, (c, d) in sorted(agg.items(), key=lambda x: -x[1][1])[:6]: print(f"{d:9.1f} us {c:4d} {k}")
PY

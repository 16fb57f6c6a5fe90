"""Per-call launch shares from an ncu --csv launch list (gpu__time_duration.sum).

    python scripts/launch_shares.py LIST.csv CALLS [--last N] [--lib]

Library (spb::) kernels only with --lib; --last N keeps the last N library
launches (the measured call of scripts/id_call.py).  Times are ncu's cold-cache,
serialised per-launch durations."""
import collections
import csv
import sys

args = sys.argv[1:]
path, calls = args[0], float(args[1])
last = int(args[args.index("--last") + 1]) if "--last" in args else 0
lib = "--lib" in args
rows = list(csv.reader(open(path)))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
data = [r for r in rows[hdr + 1:] if len(r) == len(h)]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
if lib:
    data = [r for r in data if "spb::" in r[ki]]
if last:
    data = data[-last:]
tot = collections.OrderedDict()
for r in data:
    n = r[ki].split("(")[0][:72]
    tot.setdefault(n, [0, 0.0])
    tot[n][0] += 1
    tot[n][1] += float(r[vi].replace(",", ""))
all_t = sum(t for _, t in tot.values())
print(f"# {len(data)} launches, {all_t / 1e3 / calls:.1f} us of kernel time per call ({calls:g} calls)")
print(f"# {'us/call':>9s} {'launch/call':>11s} {'share':>6s}  kernel")
for n, (c, t) in sorted(tot.items(), key=lambda x: -x[1][1])[:30]:
    print(f"  {t / 1e3 / calls:9.1f} {c / calls:11.1f} {100 * t / all_t:5.1f}%  {n}")

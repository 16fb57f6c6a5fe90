"""Per-call launch shares of a `bench.py` run from its ncu launch list
(gpu__time_duration.sum, --csv).  bench.py also launches K2 (and its Z pack,
copy2d) alone 13 times for the roofline measurement; for those two kernels the
per-call figure is one MEDIAN launch, every other kernel is total / calls.

    python scripts/bench_shares.py LIST.csv CALLS
"""
import collections
import csv
import statistics
import sys

path, calls = sys.argv[1], int(sys.argv[2])
rows = list(csv.reader(open(path)))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
per = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) != len(h) or "spb::" not in r[ki]:
        continue
    v = float(r[vi].replace(",", ""))
    v *= {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}.get(r[ui], 1e-3)
    per.setdefault(r[ki].split("(")[0][:64], []).append(v)
table = []
for name, d in per.items():
    if "skinny_tma" in name or "copy2d" in name:
        table.append((statistics.median(d), 1.0, name, len(d)))
    else:
        table.append((sum(d) / calls, len(d) / calls, name, len(d)))
tot = sum(t[0] for t in table)
print(f"# per-call sum of kernel durations: {tot:.1f} us; library launches per call: {sum(t[1] for t in table):.1f}")
print(f"# {'us/call':>9s} {'launch/call':>11s} {'share':>6s}  kernel (launches in the list)")
for us, n, name, cnt in sorted(table, reverse=True):
    print(f"  {us:9.1f} {n:11.1f} {100 * us / tot:5.1f}%  {name} ({cnt})")

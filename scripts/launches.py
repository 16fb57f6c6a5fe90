"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr]; data = [r for r in rows[hdr + 1:] if len(r) == len(h)]
ki, vi = h.index('Kernel Name'), h.index('Metric Value')
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
tot = collections.OrderedDict()
for r in data:
    n = r[ki].split('(')[0][:70]
    tot.setdefault(n, [0, 0.0]); tot[n][0] += 1; tot[n][1] += float(r[vi].replace(',', ''))
all_t = sum(t for _, t in tot.values())
print(f"{len(data)} launches, {all_t/1e3:.1f} us total, /{steps:g} steps")
for n, (c, t) in sorted(tot.items(), key=lambda x: -x[1][1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 25]:
    print(f"{t/1e3/steps:9.1f} us/step {c/steps:6.1f} launches/step  {100*t/all_t:5.1f}%  {n}")

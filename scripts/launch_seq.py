"""Print an ncu --csv launch list (gpu__time_duration.sum) in launch order."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr]; data = [r for r in rows[hdr + 1:] if len(r) == len(h)]
ki, vi = h.index('Kernel Name'), h.index('Metric Value')
lo = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3]) if len(sys.argv) > 3 else len(data)
tot = 0.0
for i, r in enumerate(data[lo:hi], lo):
    t = float(r[vi].replace(',', '')) / 1e3
    tot += t
    print(f"{i:4d} {t:8.1f} us  {tot:8.1f}  {r[ki].split('(')[0][:60]}")

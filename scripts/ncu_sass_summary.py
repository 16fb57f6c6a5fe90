"""Opcode / stall summary of one kernel from an ncu report (SASS source page).
usage: ncu_sass_summary.py REPORT LAUNCH_INDEX [top]"""
import collections, csv, io, subprocess, sys
rep, idx = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if 'Source' in r)
h = rows[hi]
si, ie = h.index('Source'), h.index('Instructions Executed')
ws = h.index('Warp Stall Sampling (All Samples)')
op, st, lines = collections.Counter(), collections.Counter(), []
for r in rows[hi + 1:]:
    if len(r) != len(h):
        continue
    toks = r[si].split()
    if not toks:
        continue
    o = toks[1] if toks[0].startswith('@') and len(toks) > 1 else toks[0]
    o = o.split('.')[0]
    try:
        n, s = float(r[ie] or 0), float(r[ws] or 0)
    except ValueError:
        continue
    op[o] += n
    st[o] += s
    lines.append((s, r[0], r[si][:70]))
tot, stot = sum(op.values()), sum(st.values()) or 1
print(f"instructions {tot:.0f}, stall samples {stot:.0f}")
for o, c in op.most_common(top):
    print(f"  {o:10s} {c:10.0f} {100 * c / tot:5.1f}%   stall {100 * st[o] / stot:5.1f}%")
print("hottest SASS lines by stall samples:")
for s, a, src in sorted(lines, reverse=True)[:top]:
    print(f"  {100 * s / stot:5.1f}%  {a}  {src}")

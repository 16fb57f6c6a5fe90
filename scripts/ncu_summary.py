"""Key metrics of an ncu --set full report (read here, no GPU needed)."""
import csv, subprocess, sys
WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'launch__grid_size', 'launch__block_size', 'launch__registers_per_thread', 'smsp__inst_executed.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'sm__cycles_elapsed.avg.per_second',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active']
STALLS = 'smsp__average_warps_issue_stalled_'
for rep in sys.argv[1:]:
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    for v in rows[2:]:
        print('==', rep, v[h.index('Kernel Name')][:80] if 'Kernel Name' in h else '')
        for w in WANT:
            if w in h:
                print(f'  {w:70s} {v[h.index(w)]} {units[h.index(w)]}')
        st = []
        for i in range(len(h)):
            if h[i].startswith(STALLS) and h[i].endswith('_per_issue_active.ratio') and v[i]:
                try:
                    st.append((float(v[i]), h[i][len(STALLS):]))
                except ValueError:
                    pass
        print('  stalls:', ', '.join(f'{n.replace("_per_issue_active.ratio","")}={x:.2f}'
                                    for x, n in sorted(st, reverse=True)[:6]))

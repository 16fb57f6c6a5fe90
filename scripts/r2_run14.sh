timeout 600 python scripts/bj_timeline.py 1500 1100 2>/dev/null | head -7
timeout 600 python scripts/bj_timeline.py 5000 4096 2>/dev/null | head -10
timeout 600 python scripts/bj_probe.py 2>&1 | tail -3

timeout 600 python scripts/bj_probe.py 2>&1 | tail -4
timeout 600 python scripts/bj_timeline.py 5000 4096 2>/dev/null | head -10

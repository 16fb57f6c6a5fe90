timeout 600 python scripts/bj_timeline.py 1500 1100 2>/dev/null | head -10

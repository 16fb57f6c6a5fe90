timeout 600 python scripts/bj_timeline.py 5000 4096
timeout 600 python scripts/bj_timeline.py 2000 20000 | head -8
timeout 900 python scripts/id_call.py cfg5 2>&1 | tail -2
timeout 600 python scripts/id_timeline.py cfg5 | head -12

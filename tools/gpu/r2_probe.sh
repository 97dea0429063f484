timeout 600 python tools/rank_probe.py 8 2>&1 | tail -12

timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python tools/moe_time.py 2>&1 | tail -12

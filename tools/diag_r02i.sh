timeout 300 python tools/time_route3.py 2>&1 | head -22

SPECSV_ROUTE3_FORCE_EXACT=1 timeout 300 python tools/time_route3.py 2>&1 | tail -22

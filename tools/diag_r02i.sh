for f in 0 4 0 4; do echo "== $f"; SPECSV_ROUTE3_DEBUG=$f timeout 300 python tools/time_route3.py 2>&1 | grep -E "route3_kernel|selected|select:"; done

# route3 phases + step numbers
python tools/time_route3.py 2>&1 | tail -16
for i in 1 2 3; do timeout 600 python bench.py --steps 30 --warmup 5 --skip-cpu-baseline --skip-decode-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1), round(d['detail']['route_us_per_launch'],2), round(d['detail']['attend_us_per_launch'],2))"; done

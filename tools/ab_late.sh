# refresh-layer late splits: default (skip 2) vs off (SPECSV_ATTEND_LATE_SKIP=0) vs skip 3
for v in 2 0 3 2 0 3; do
  SPECSV_ATTEND_LATE_SKIP=$v timeout 600 python bench.py --steps 30 --warmup 5 --skip-cpu-baseline --skip-decode-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('late_skip=$v', round(d['value'],1), round(d['e2e']['value'],1), round(d['detail']['attend_us_per_launch'],2))"
done

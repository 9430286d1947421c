# same-box A/B of the attend split count (SPECSV_ATTEND_SPLITS) under the early trigger
for v in 18 16 14 12 18 16 14 12; do
  SPECSV_ATTEND_SPLITS=$v timeout 600 python bench.py --steps 30 --warmup 5 --skip-cpu-baseline --skip-decode-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('splits=$v', round(d['value'],1), round(d['e2e']['value'],1), round(d['detail']['attend_us_per_launch'],2))"
done

# split CTAs per head (SPECSV_ATTEND_SPLITS caps them)
for sp in 18 16 17 18 16 17; do
  SPECSV_ATTEND_SPLITS=$sp timeout 600 python bench.py --steps 30 --warmup 5 --skip-cpu-baseline --skip-decode-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('splits=$sp', round(d['value'],1), round(d['e2e']['value'],1), round(d['detail']['attend_us_per_launch'],2))"
done

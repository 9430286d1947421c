# same-box A/B of one SPECSV_ROUTE3_DEBUG bit: bash tools/ab_route_flag.sh <bit value>
for v in 0 $1 0 $1 0 $1; do
  SPECSV_ROUTE3_DEBUG=$v timeout 600 python bench.py --steps 30 --warmup 5 --skip-cpu-baseline --skip-decode-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('route3 debug=$v', round(d['value'],1), round(d['e2e']['value'],1), round(d['detail']['route_us_per_launch'],2), round(d['detail']['attend_us_per_launch'],2))"
done

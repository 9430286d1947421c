# same-box A/B of the refresh layers' attend split count (SPECSV_ATTEND_SPLITS_REFRESH):
# the routing launch's Top-n CTAs hold 9 SMs while the refresh attend grid is placed
for v in 0 17 16 0 17 16 0 17 16; do
  SPECSV_ATTEND_SPLITS_REFRESH=$v timeout 600 python bench.py --steps 30 --warmup 5 --skip-cpu-baseline --skip-decode-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('splits_refresh=$v', round(d['value'],1), round(d['e2e']['value'],1), round(d['detail']['attend_us_per_launch'],2))"
done

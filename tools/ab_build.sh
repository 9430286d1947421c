# same-box A/B of the default build against the per-tile-stamp diagnostics build
b() { timeout 600 python bench.py --steps 30 --warmup 5 --skip-cpu-baseline --skip-decode-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value'],1), round(d['e2e']['value'],1), round(d['detail']['attend_us_per_launch'],2))"; }
for i in 1 2; do
  python -m paper_2605_19893_b200.build --force > /dev/null 2>&1; b default
  SPECSV_TRACE_TILES=1 python -m paper_2605_19893_b200.build --force > /dev/null 2>&1; b tile_stamps
done
python -m paper_2605_19893_b200.build --force > /dev/null 2>&1

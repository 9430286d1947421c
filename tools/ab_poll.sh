# A/B: TMA producer polling with a 20 ns sleep between empty polls (SPECSV_ATTEND_DEBUG=128) vs a tight spin
for v in 0 128; do SPECSV_ATTEND_DEBUG=$v TRACE_TILES=1 python tools/trace_step.py 2 2>&1 | grep -A9 "layer  1" | grep -v "gcd\|tile 3"; done
for v in 0 128 0 128; do
  SPECSV_ATTEND_DEBUG=$v timeout 600 python bench.py --steps 20 --warmup 5 --skip-cpu-baseline --skip-decode-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('debug=$v', d['value'], d['e2e']['value'], d['detail']['attend_us_per_launch'])"
done

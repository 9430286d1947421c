SPECSV_ATTEND_DEBUG=32 TRACE_TILES=1 timeout 120 python tools/trace_step.py 4 2>&1 | grep "check"
TRACE_TILES=1 timeout 120 python tools/trace_step.py 2 2>&1 | grep -A8 "layer  "
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 --skip-cpu-baseline --skip-decode-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['detail']['route_us_per_launch'], d['detail']['attend_us_per_launch'])"; done

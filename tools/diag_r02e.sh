timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "route_kernels or c4_shape or batched or refresh_then_reuse" > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
timeout 300 python tools/time_route3.py 2>&1 | head -12
timeout 600 python bench.py --steps 20 --warmup 5 --skip-cpu-baseline --skip-decode-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['detail']['route_us_per_launch'], d['detail']['attend_us_per_launch'])"

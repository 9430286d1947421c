timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
timeout 600 python tools/trace_step.py 4 2>&1 | head -5
timeout 600 python bench.py --steps 20 --warmup 5 --skip-cpu-baseline --skip-decode-baseline > gpurun_out/b.json 2>gpurun_out/b.err; head -c 150 gpurun_out/b.json

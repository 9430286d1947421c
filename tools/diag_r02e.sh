timeout 600 python tools/trace_step.py 4 2>&1 | head -5
timeout 600 python bench.py --steps 20 --warmup 5 --skip-cpu-baseline --skip-decode-baseline > gpurun_out/b.json 2>gpurun_out/b.err; head -c 200 gpurun_out/b.json

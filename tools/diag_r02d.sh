set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gt.log 2>&1; tail -3 gpurun_out/gt.log
timeout 900 python bench.py --steps 20 --warmup 5 --skip-cpu-baseline --skip-decode-baseline > gpurun_out/b.json 2> gpurun_out/b.err; head -c 300 gpurun_out/b.json
timeout 600 python tools/trace_step.py 4 > gpurun_out/trace_step.txt 2>&1; cat gpurun_out/trace_step.txt

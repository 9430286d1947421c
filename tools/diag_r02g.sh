timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gt.log 2>&1; tail -2 gpurun_out/gt.log
timeout 600 python tools/trace_step.py 4 2>&1 | head -5
timeout 300 python tools/time_route3.py 2>&1 | tail -20

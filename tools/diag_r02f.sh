timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "route_kernels or refresh_then_reuse or c4 or deterministic or batched" > gpurun_out/t_route.log 2>&1; tail -3 gpurun_out/t_route.log
timeout 300 python tools/time_route3.py > gpurun_out/route3b.txt 2>&1; head -2 gpurun_out/route3b.txt
timeout 600 python tools/trace_step.py 4 > gpurun_out/trace_step.txt 2>&1; cat gpurun_out/trace_step.txt

set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "digit_planes or route_kernels or refresh_then_reuse or c3 or c4 or c5" > gpurun_out/t_route.log 2>&1; tail -15 gpurun_out/t_route.log
timeout 300 python tools/time_route3.py > gpurun_out/route3b.txt 2>&1; cat gpurun_out/route3b.txt

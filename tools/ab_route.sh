# quick A/B of the routing kernel: timeline, timing, parity of the routing-heavy tests
python tools/trace_route.py > gpurun_out/tr.log 2>&1
python tools/time_route.py >> gpurun_out/tr.log 2>&1
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2 > gpurun_out/ab_tests.txt

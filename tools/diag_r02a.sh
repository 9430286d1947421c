set -x
timeout 600 python tools/time_route3.py > gpurun_out/route3.txt 2>&1
timeout 600 python tools/trace_step.py 4 > gpurun_out/trace_step.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k c4_shape > gpurun_out/c4shape.log 2>&1; tail -3 gpurun_out/c4shape.log

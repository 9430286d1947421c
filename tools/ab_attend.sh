# quick A/B of the verify step: bench without the CPU / decode legs, attend trace
python bench.py --steps 20 --warmup 5 --skip-cpu-baseline --skip-decode-baseline > gpurun_out/ab.log 2>&1
python tests/debug_run.py 65536 8 trace > gpurun_out/ta.log 2>&1
python -m pytest tests/test_gpu_parity.py -x -q -k "verify" 2>&1 | tail -2 > gpurun_out/ab_tests.txt

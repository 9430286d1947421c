# repeat the GPU parity suite, keeping the first failure's report
for i in 1 2 3 4; do
  python -m pytest tests/test_gpu_parity.py -q -p no:randomly > gpurun_out/flake_$i.txt 2>&1
  tail -1 gpurun_out/flake_$i.txt
done

T='tests/test_gpu_parity.py::test_verify_other_nsa_configs'
for env in "X=0" "SPECSV_ROUTE3_DEBUG=32" "SPECSV_ROUTE_LEGACY=1" "SPECSV_ROUTE3_FORCE_EXACT=1"; do
  echo "== $env"; env $env timeout 300 python -m pytest "$T" -m gpu -q -k "4" 2>&1 | grep -E "passed|failed|gap" | head -4
done > gpurun_out/n48.txt 2>&1

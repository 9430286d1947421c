# Top-n selection with 8-lane groups and compacted survivor scores vs the
# earlier form (SPECSV_ROUTE3_DEBUG=32): GPU tests, same-box step A/B, and the
# select cycle counts of the diagnostics build
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gt.log 2>&1; tail -3 gpurun_out/gt.log
SPECSV_ROUTE3_DEBUG=32 timeout 900 python -m pytest tests/test_gpu_parity_c3.py -m gpu -x -q > gpurun_out/gt_old.log 2>&1; tail -2 gpurun_out/gt_old.log
bash tools/ab_route_flag.sh 32 > gpurun_out/ab_select.txt 2>&1
SPECSV_TRACE_TILES=1 python -m paper_2605_19893_b200.build --force > /dev/null 2>&1
timeout 300 python tools/time_route3.py > gpurun_out/route3_new.txt 2>&1
SPECSV_ROUTE3_DEBUG=32 timeout 300 python tools/time_route3.py > gpurun_out/route3_old.txt 2>&1
python -m paper_2605_19893_b200.build --force > /dev/null 2>&1

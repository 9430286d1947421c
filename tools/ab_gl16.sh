# Top-n selection in groups of 16 lanes (n <= 32) vs the earlier form
# (SPECSV_ROUTE3_DEBUG=32): parity tests (n = 48 covers the 8-lane groups),
# same-box step A/B, select cycles of the diagnostics build
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gt.log 2>&1; tail -1 gpurun_out/gt.log
bash tools/ab_route_flag.sh 32 > gpurun_out/ab_gl16.txt 2>&1
SPECSV_TRACE_TILES=1 python -m paper_2605_19893_b200.build --force > /dev/null 2>&1
timeout 300 python tools/time_route3.py > gpurun_out/route3_gl16.txt 2>&1
python -m paper_2605_19893_b200.build --force > /dev/null 2>&1

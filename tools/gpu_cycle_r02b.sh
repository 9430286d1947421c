# one full measurement cycle on a B200 box: GPU tests, smoke, bench, reference arm,
# launch list, ncu captures of the attend and routing kernels
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gt.log 2>&1; tail -3 gpurun_out/gt.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/b.json 2> gpurun_out/b.err; cat gpurun_out/b.json | head -c 600
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref.json 2> gpurun_out/ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch.csv python bench.py --steps 2 --warmup 3 --skip-decode-baseline --skip-cpu-baseline > /dev/null 2>&1
timeout 600 ncu -k regex:nsa_attend --launch-skip 2 --launch-count 1 --set full --clock-control none --import-source on -f -o gpurun_out/attend python tools/prof_attend.py > gpurun_out/pa.log 2>&1
timeout 600 ncu -k regex:route3 --launch-skip 2 --launch-count 1 --set full --clock-control none --import-source on -f -o gpurun_out/route python tools/prof_route.py > gpurun_out/pr.log 2>&1
# the timelines need the diagnostics build (trace stamps compiled in)
SPECSV_TRACE_TILES=1 python -m paper_2605_19893_b200.build --force > /dev/null 2>&1
TRACE_TILES=1 timeout 600 python tools/trace_step.py 4 > gpurun_out/trace_step.txt 2>&1
timeout 300 python tools/time_route3.py > gpurun_out/route3.txt 2>&1
python -m paper_2605_19893_b200.build --force > /dev/null 2>&1

bash tools/c4_runs.sh

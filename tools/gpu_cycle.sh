set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/gt.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch.csv python bench.py --steps 2 --warmup 1 --skip-decode-baseline > /dev/null 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/b.log 2> gpurun_out/bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref.log 2> gpurun_out/ref.err
ncu -k regex:nsa_attend --launch-skip 2 --launch-count 1 --set full --clock-control none --import-source on -f -o gpurun_out/attend python tools/prof_attend.py > gpurun_out/pa.log 2>&1
ncu -k regex:route_fused --launch-skip 2 --launch-count 1 --set full --clock-control none --import-source on -f -o gpurun_out/route python tools/prof_route.py > gpurun_out/pr.log 2>&1
ls -la gpurun_out

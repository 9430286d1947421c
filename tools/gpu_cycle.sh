# one GPU round trip: gpu tests, ncu launch list of a short bench, then the bench
python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/gt.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch.csv python bench.py --steps 2 --warmup 1 > /dev/null 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/b.log 2> gpurun_out/bench.err

set -x
timeout 600 ncu -k regex:route3 --launch-skip 2 --launch-count 1 --set full --import-source on --clock-control none -f -o gpurun_out/route3 python tools/prof_route.py > gpurun_out/pr3.log 2>&1
ncu -i gpurun_out/route3.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/route3_src.csv 2>/dev/null
ls -la gpurun_out/route3*

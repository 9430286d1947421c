timeout 600 ncu -k regex:nsa_attend --launch-skip 2 --launch-count 1 --set full --import-source on --clock-control none -f -o gpurun_out/attend_r02 python tools/prof_attend.py > gpurun_out/pa.log 2>&1
ncu -i gpurun_out/attend_r02.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/attend_src.csv 2>/dev/null
ls -la gpurun_out/attend_r02*

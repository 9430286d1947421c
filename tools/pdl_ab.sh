set -x
timeout 600 python bench.py --steps 10 --warmup 3 --skip-cpu-baseline --skip-decode-baseline > gpurun_out/b_pdl.json 2> gpurun_out/b_pdl.err
SPECSV_NO_PDL=1 timeout 600 python bench.py --steps 10 --warmup 3 --skip-cpu-baseline --skip-decode-baseline > gpurun_out/b_nopdl.json 2> gpurun_out/b_nopdl.err
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gt6.log 2>&1; tail -3 gpurun_out/gt6.log

# A/B: attend launched cooperative vs placed early under PDL (bench C2)
set -x
timeout 600 python bench.py --steps 20 --warmup 5 --skip-cpu-baseline --skip-decode-baseline > gpurun_out/b_nocoop.json 2> gpurun_out/b_nocoop.err
SPECSV_ATTEND_COOP=1 timeout 600 python bench.py --steps 20 --warmup 5 --skip-cpu-baseline --skip-decode-baseline > gpurun_out/b_coop.json 2> gpurun_out/b_coop.err
SPECSV_ROUTE3=1 timeout 600 python bench.py --steps 20 --warmup 5 --skip-cpu-baseline --skip-decode-baseline > gpurun_out/b_r3.json 2> gpurun_out/b_r3.err

# the last K split arrivals of a head merge it (SPECSV_ATTEND_MERGERS=K), the
# others exit after their partials: GPU tests at K=6 and the default, step A/B
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gt.log 2>&1; tail -1 gpurun_out/gt.log
SPECSV_ATTEND_MERGERS=6 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pdl_chain.py tests/test_gpu_parity_c3.py -m gpu -x -q > gpurun_out/gt_k6.log 2>&1; tail -1 gpurun_out/gt_k6.log
for v in 0 9 6 4 0 9 6 4; do
  SPECSV_ATTEND_MERGERS=$v timeout 600 python bench.py --steps 30 --warmup 5 --skip-cpu-baseline --skip-decode-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mergers=$v', round(d['value'],1), round(d['e2e']['value'],1), round(d['detail']['attend_us_per_launch'],2))"
done > gpurun_out/ab_mergers.txt 2>&1; cat gpurun_out/ab_mergers.txt
for v in 0 6; do
  SPECSV_ATTEND_MERGERS=$v timeout 900 python bench.py --ctx 131072 --layers 4 --requests 8 --steps 10 --warmup 3 --skip-cpu-baseline --skip-decode-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 r8 mergers=$v', round(d['value'],1), round(d['e2e']['value'],1))"
done >> gpurun_out/ab_mergers.txt 2>&1
SPECSV_NO_PDL=1 SPECSV_ATTEND_MERGERS=0 timeout 600 python bench.py --steps 20 --warmup 5 --skip-cpu-baseline --skip-decode-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nopdl mergers=0', round(d['value'],1), round(d['detail']['attend_us_per_launch'],2))" >> gpurun_out/ab_mergers.txt 2>&1
SPECSV_NO_PDL=1 SPECSV_ATTEND_MERGERS=6 timeout 600 python bench.py --steps 20 --warmup 5 --skip-cpu-baseline --skip-decode-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nopdl mergers=6', round(d['value'],1), round(d['detail']['attend_us_per_launch'],2))" >> gpurun_out/ab_mergers.txt 2>&1

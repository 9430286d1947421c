# route3: Top-n arrival atomic relaxed and overlapped with the score-row loads
# vs acq_rel before them (SPECSV_ROUTE3_DEBUG=128)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gt.log 2>&1; tail -1 gpurun_out/gt.log
bash tools/ab_route_flag.sh 128 > gpurun_out/ab_cnt_overlap.txt 2>&1; cat gpurun_out/ab_cnt_overlap.txt
for v in 0 128; do
  SPECSV_ROUTE3_DEBUG=$v timeout 900 python bench.py --ctx 131072 --layers 4 --requests 8 --steps 10 --warmup 3 --skip-cpu-baseline --skip-decode-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 r8 route3 debug=$v', round(d['value'],1), round(d['e2e']['value'],1))"
done >> gpurun_out/ab_cnt_overlap.txt 2>&1

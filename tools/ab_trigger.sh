# early PDL trigger in the attend kernel (after the tile loop) vs the old late
# trigger (after the merge, SPECSV_ATTEND_DEBUG=256): GPU tests, same-box A/B,
# the C4 batched line, and the step timeline of the diagnostics build
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gt.log 2>&1; tail -3 gpurun_out/gt.log
bash tools/ab_flag.sh 256 > gpurun_out/ab_trigger.txt 2>&1; cat gpurun_out/ab_trigger.txt
for v in 0 256; do
  SPECSV_ATTEND_DEBUG=$v timeout 600 python bench.py --gpus 1 --workload c4 --steps 10 --warmup 3 --skip-cpu-baseline --skip-decode-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 debug=$v', round(d['value'],1), round(d['e2e']['value'],1))"
done > gpurun_out/ab_trigger_c4.txt 2>&1; cat gpurun_out/ab_trigger_c4.txt
SPECSV_TRACE_TILES=1 python -m paper_2605_19893_b200.build --force > /dev/null 2>&1
timeout 600 python tools/trace_step.py 4 > gpurun_out/trace_step.txt 2>&1
SPECSV_ATTEND_DEBUG=256 timeout 600 python tools/trace_step.py 4 > gpurun_out/trace_step_late.txt 2>&1
python -m paper_2605_19893_b200.build --force > /dev/null 2>&1

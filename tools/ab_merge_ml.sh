# split merge: one (m, l) load per lane, shuffled out, vs every thread loading
# every split's (m, l) (SPECSV_ATTEND_DEBUG=1024): GPU tests, same-box A/B
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gt.log 2>&1; tail -1 gpurun_out/gt.log
bash tools/ab_flag.sh 1024 > gpurun_out/ab_merge_ml.txt 2>&1; cat gpurun_out/ab_merge_ml.txt

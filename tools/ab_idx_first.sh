# REUSE index rows staged before the CTA-wide barrier (ahead of the compressed
# stages' TMA burst) vs after it (SPECSV_ATTEND_DEBUG=512): GPU tests, same-box A/B
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gt.log 2>&1; tail -1 gpurun_out/gt.log
bash tools/ab_flag.sh 512 > gpurun_out/ab_idx_first.txt 2>&1; cat gpurun_out/ab_idx_first.txt

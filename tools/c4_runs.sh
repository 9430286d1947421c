# C4: 128K context, 4 layer caches per request, gamma=8 chain, exact C=4,
# alt schedule; the per-GPU request counts of 64 requests over 8 / 4 / 2 GPUs
for R in 8 16 32; do
  timeout 900 python bench.py --ctx 131072 --layers 4 --requests $R --steps 10 --warmup 3 \
      --skip-cpu-baseline --skip-decode-baseline > gpurun_out/c4_r$R.json 2> gpurun_out/c4_r$R.err
done

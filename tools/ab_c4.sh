# C4 A/B: batched attend with / without the cooperative attribute (SPECSV_ATTEND_COOP=1 keeps it)
for v in 0 1 0 1; do
  if [ $v = 1 ]; then export SPECSV_ATTEND_COOP=1; else unset SPECSV_ATTEND_COOP; fi
  timeout 900 python bench.py --ctx 131072 --layers 4 --requests 8 --steps 10 --warmup 3 --skip-cpu-baseline --skip-decode-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('coop=$v', round(d['value'],1), round(d['e2e']['value'],1), round(d['ms_per_step']*1e3,1))"
done

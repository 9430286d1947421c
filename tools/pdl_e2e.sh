for v in 0 1 0 1; do
  if [ $v = 1 ]; then export SPECSV_NO_PDL=1; else unset SPECSV_NO_PDL; fi
  timeout 600 python bench.py --steps 30 --warmup 5 --skip-cpu-baseline --skip-decode-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('no_pdl=$v', round(d['value'],1), round(e['value'],1), round(e['ms_per_step']*1e3,1), round(d['ms_per_step']*1e3,1))"
done

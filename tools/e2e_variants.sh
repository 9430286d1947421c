# e2e diagnostics: drop one part of the advancing step at a time
for v in "" nocommit nocopy nod2h; do
  SPECSV_E2E_VARIANT=$v timeout 600 python bench.py --steps 30 --warmup 5 --skip-cpu-baseline --skip-decode-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('variant=$v', round(d['value'],1), round(e['value'],1), round(e['ms_per_step']*1e3,1), 'us/step; host', {k: round(x,1) for k,x in e['host_us_per_step'].items()})"
done

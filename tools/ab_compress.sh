N=compress
b() { timeout 600 python bench.py --steps 30 --warmup 5 --skip-cpu-baseline --skip-decode-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value'],1), round(d['e2e']['value'],1), round(d['e2e']['ms_per_step']*1e3,1))"; }
F=paper_2605_19893_b200/csrc/$N.cu
cp $F /tmp/new.cu
for i in 1 2; do
  cp /tmp/new.cu $F; python -m paper_2605_19893_b200.build > /dev/null 2>&1; b new
  cp .ab/${N}_base.cu $F; python -m paper_2605_19893_b200.build > /dev/null 2>&1; b base
done
cp /tmp/new.cu $F; python -m paper_2605_19893_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "compress or commit" 2>&1 | tail -2

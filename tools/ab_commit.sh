b() { timeout 600 python bench.py --steps 30 --warmup 5 --skip-cpu-baseline --skip-decode-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value'],1), round(d['e2e']['value'],1), round(d['e2e']['ms_per_step']*1e3,1))"; }
for N in compress draft_tree; do cp paper_2605_19893_b200/csrc/$N.cu /tmp/new_$N.cu; done
for i in 1 2; do
  for N in compress draft_tree; do cp /tmp/new_$N.cu paper_2605_19893_b200/csrc/$N.cu; done
  python -m paper_2605_19893_b200.build > /dev/null 2>&1; b new
  for N in compress draft_tree; do cp .ab/${N}_base.cu paper_2605_19893_b200/csrc/$N.cu; done
  python -m paper_2605_19893_b200.build > /dev/null 2>&1; b base
done
for N in compress draft_tree; do cp /tmp/new_$N.cu paper_2605_19893_b200/csrc/$N.cu; done
python -m paper_2605_19893_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "compress or commit or lossless" 2>&1 | tail -2

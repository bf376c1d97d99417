# A/B on one box: the session-start kernel (_ab_old, commit 968615b) vs HEAD, interleaved
for r in 1 2 3; do
  (cd _ab_old && timeout 600 python bench.py --no-sweep --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('OLD', round(d['value'],1), round(d['roofline']['frac'],3))")
  timeout 600 python bench.py --no-sweep --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('NEW', round(d['value'],1), round(d['roofline']['frac'],3))"
  DASH_NO_PREFETCH=1 timeout 600 python bench.py --no-sweep --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('NEW-nopf', round(d['value'],1), round(d['roofline']['frac'],3))"
done
for s in 2048,16384; do
  (cd _ab_old && timeout 300 python scripts/exp_reduce_path.py $s 128 causal | sed 's/^/OLD /')
  timeout 300 python scripts/exp_reduce_path.py $s 128 causal | sed 's/^/NEW /'
done

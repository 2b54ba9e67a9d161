python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for cfg in C5 C1; do
timeout 300 python bench.py --config $cfg --steps 50 --warmup 5 2>&1 | tail -1 > gpurun_out/bench_$cfg.json
python -c "import json; d=json.load(open('gpurun_out/bench_$cfg.json')); print('$cfg', d['value'], (d.get('e2e') or {}).get('value'), d.get('passes'))"
done

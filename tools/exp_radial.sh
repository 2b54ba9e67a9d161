python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for cfg in C2 C3 C5; do
timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --e2e-steps 0 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$cfg', d['value'], d.get('passes'))"
done

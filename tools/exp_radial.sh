python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for s in 4 1; do
TLSPH_BSPLIT=$s timeout 300 python bench.py --config C4 --steps 50 --warmup 5 --e2e-steps 0 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('C4 split$s', d['value'], d.get('passes'))"
done

for v in "TLSPH_HALO_CAP=1.0" "TLSPH_HALO_CAP=1.3" "TLSPH_HALO_RESIDUE=1"; do
for cfg in C2 C3; do
env $v timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --e2e-steps 0 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$cfg $v', round(d['value']/1e9,3), d['passes']['pass_a_ms'], d['passes']['pass_b_ms'])"
done
done

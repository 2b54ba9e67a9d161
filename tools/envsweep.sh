#!/bin/bash
# usage: tools/envsweep.sh [--config C4] [--precision fp32] "ENV=a ENV2=b" "ENV=c" ...
# one short bench line per environment setting (step rate, per-pass ms and roofline fractions)
cfg=C4; prec=fp32
while [[ "$1" == --* ]]; do
  case "$1" in --config) cfg=$2; shift 2;; --precision) prec=$2; shift 2;; esac
done
for e in "$@"; do
  env $e python bench.py --config $cfg --precision $prec --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-fp64 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); p=d['passes']
print('$cfg $prec [$e]', round(d['value']/1e9,3),'G/s', 'A',round(p['pass_a_ms'],3),'ms',round(p['frac_a'],3),'B',round(p['pass_b_ms'],3),'ms',round(p['frac_b'],3))" || echo "$e failed"
done

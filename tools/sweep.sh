#!/bin/bash
# usage: tools/sweep.sh lib1 lib2 ... : FP32 + FP64 bench lines per library variant
for lib in "$@"; do
  for prec in fp32 fp64; do
    TLSPH_LIB=$PWD/paper_2602_15149_b200/$lib python bench.py --steps 10 --warmup 3 --precision $prec --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); p=d['passes']
print('$lib $prec', round(d['value']/1e9,3),'G/s', 'A',round(p['pass_a_ms'],3),'ms',round(p['frac_a'],3),'B',round(p['pass_b_ms'],3),'ms',round(p['frac_b'],3))"
  done
done

#!/bin/bash
# One default bench line per BASELINE config (the driver's command with
# --config), written to gpurun_out/<tag>_bench_<cfg>.json; copy the ones to
# keep into profiles/.   usage: tools/bench_all.sh <tag> [configs...]
tag=${1:-rX}; shift
cfgs=${@:-C1 C2 C3 C4 C5 P1}
for c in $cfgs; do
  timeout 1200 python bench.py --config $c > gpurun_out/${tag}_bench_$c.log 2>&1
  grep '^{' gpurun_out/${tag}_bench_$c.log | tail -1 > gpurun_out/${tag}_bench_$c.json
  python -c "
import json; d=json.load(open('gpurun_out/${tag}_bench_$c.json')); p=d['passes']
print('$c', round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],4), 'ms/step', 'A', round(p['pass_a_ms'],3), 'B', round(p['pass_b_ms'],3), 'fp64', round(d['fp64']['value']/1e9,3), 'e2e', round(d['e2e']['value']/1e9,3), d['clocks'])" || echo "$c failed"
done

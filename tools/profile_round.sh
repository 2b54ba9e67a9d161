#!/bin/bash
# GPU-side profiling of the bench workload (run under gpurun):
#   1. launch list of the timed steps (per-launch durations, serialised)
#   2. one `ncu --set full` capture of pass A and pass B, exported to CSV
#      (tools/ncu_box.sh; read here with tools/ncu_report.py / stall_lines.py)
# Outputs land in gpurun_out/$1_*; summarise into profiles/ with
# tools/launch_summary.py and tools/ncu_report.py.
tag=${1:-prof}
cfg=${2:-C4}
kre=${3:-k_pass}
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-fp64 \
    > gpurun_out/${tag}_launch.log 2>&1
tools/ncu_box.sh ${tag}_full $kre 8 2 ${kre}_a ${kre}_b -- \
    python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-fp64
tail -1 gpurun_out/${tag}_launch.log | cut -c1-200

#!/bin/bash
# GPU-side profiling of the bench workload (run under gpurun):
#   1. launch list of the timed steps (per-launch durations, serialised)
#   2. one `ncu --set full` capture of pass A and pass B
# Outputs land in gpurun_out/$1_*; summarise here with tools/launch_summary.py
# and tools/ncu_report.py into profiles/.
tag=${1:-prof}
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pass -s 8 -c 2 \
    -o gpurun_out/${tag}_full \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_full.log 2>&1
tail -1 gpurun_out/${tag}_launch.log | cut -c1-200

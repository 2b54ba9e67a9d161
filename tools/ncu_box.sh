#!/bin/bash
# GPU-box side: one `ncu --set full` capture, exported to gzipped CSVs that
# fit gpurun's copy-back limit (tools/ncu_io.py reads them).
#   tools/ncu_box.sh <out-name> <kernel-regex> <skip> <count> <src-regex...> -- <command...>
name=$1; kre=$2; skip=$3; cnt=$4; shift 4
srcs=()
while [[ "$1" != "--" ]]; do srcs+=("$1"); shift; done
shift
rep=gpurun_out/$name.ncu-rep
ncu --set full --clock-control none --import-source on -k regex:$kre -s $skip -c $cnt -o ${rep%.ncu-rep} "$@" > gpurun_out/$name.log 2>&1
ncu -i $rep --page raw --csv | gzip > $rep.raw.csv.gz
for s in "${srcs[@]}"; do
  ncu -i $rep --page source --csv --print-source sass -k regex:$s | gzip > $rep.src.$s.csv.gz
done
rm -f $rep
ls -la gpurun_out/$name*

#!/bin/bash
# Launch list + ncu --set full captures of the top kernels of one cfg3 step (run under gpurun).
# Usage: bash tools/gpu_profile.sh <tag> [kernel regex ...]
tag=${1:-prof}; shift
out=gpurun_out/$tag; mkdir -p $out
export HODLR_ACA_NOGRAPH=1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python tools/prof_step.py cfg3 1 > $out/launches.log 2>&1
for spec in "$@"; do
  k=${spec%%:*}; skip=${spec#*:}; [ "$skip" = "$spec" ] && skip=0
  timeout 400 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip $skip -c 1 \
    -o $out/$k python tools/prof_step.py cfg3 1 > $out/$k.log 2>&1
  ncu -i $out/$k.ncu-rep --page details --csv > $out/$k.details.csv 2>/dev/null
done
ls -la $out

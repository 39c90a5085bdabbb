#!/bin/bash
# Round evidence (run under gpurun): bench JSON line, ncu launch list of one bench-config step, and
# ncu --set full captures of the main kernels with their summaries.  bash tools/round_profile.sh <tag>
tag=${1:-r01}; out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/gpu.txt
timeout 600 python bench.py --steps 5 --warmup 3 > $out/bench.json 2> $out/bench.err || tail -20 $out/bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_reference.json 2>> $out/bench.err
HODLR_ACA_NOGRAPH=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/launches.csv python tools/prof_step.py cfg3 1 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/launches_graph.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
for spec in k_aca_pass:12 k_leaf_zsyrk:0 k_leaf_chol:0 k_tree_factor:0 k_solve:0 k_aca_fused:0; do
  k=${spec%%:*}; skip=${spec#*:}
  HODLR_ACA_NOGRAPH=1 timeout 400 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip $skip -c 1 \
    -o $out/$k python tools/prof_step.py cfg3 1 > $out/$k.log 2>&1
  ncu -i $out/$k.ncu-rep --page raw --csv > $out/$k.raw.csv 2>/dev/null
done
python tools/ncu_summary.py $out "${2:-1}" "ncu --set full --clock-control none, one launch each (tools/round_profile.sh, cfg3 n=2^20 step)" || true
ls $out

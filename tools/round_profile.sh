#!/bin/bash
# Round evidence (run under gpurun): bench JSON lines (own arm + reference arm), ncu launch lists of one bench-config
# step (graph and host-loop ACA), the per-family DRAM traffic of one step, ncu --set full captures of the main
# kernels with their summaries, all five configurations, the batched config-4 sweep and the scaling projection.
#   bash tools/round_profile.sh <tag>
tag=${1:-r02}; out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)" > $out/cpu.txt
HODLR_ACA_NOGRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $out/traffic.csv python tools/prof_step.py cfg3 1 > /dev/null 2>&1
python tools/ncu_traffic.py $out/traffic.csv $out/traffic.json && cp $out/traffic.json profiles/${tag}_traffic.json
timeout 600 python bench.py --steps 5 --warmup 3 > $out/bench.json 2> $out/bench.err || tail -20 $out/bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_reference.json 2>> $out/bench.err
HODLR_ACA_NOGRAPH=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/launches.csv python tools/prof_step.py cfg3 1 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/launches_graph.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
for spec in k_aca_pass:24 k_leaf_zsyrk:0 k_leaf_chol:0 k_tree_deep:0 k_tree_top:0 k_solve:0 k_aca_fused:0; do
  k=${spec%%:*}; skip=${spec#*:}
  HODLR_ACA_NOGRAPH=1 timeout 400 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip $skip -c 1 \
    -o $out/$k python tools/prof_step.py cfg3 1 > $out/$k.log 2>&1
  ncu -i $out/$k.ncu-rep --page raw --csv > $out/$k.raw.csv 2>/dev/null
done
python tools/ncu_summary.py $out "${2:-2}" "ncu --set full --clock-control none, one launch each (tools/round_profile.sh, cfg3 n=2^20 step)" || true
cp profiles/r0${2:-2}_* $out/ 2>/dev/null
timeout 900 python tools/all_configs.py $out/configs.json > $out/configs.log 2>&1 || tail -5 $out/configs.log
timeout 300 python tools/sweep_bench.py 5 > $out/sweep.log 2>&1 || tail -5 $out/sweep.log
timeout 600 python tools/project_scaling.py cfg3 $out/scaling_projection.json > $out/scaling.log 2>&1 || tail -5 $out/scaling.log
rm -f $out/*.ncu-rep
ls $out

#!/bin/bash
# GPU check used during development: parity tests, bench, launch list (run under gpurun).
tag=${1:-q}; out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > $out/pytest_gpu.log; tail -3 $out/pytest_gpu.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $out/bench.json 2> $out/bench.err
python -c "import json; d=json.load(open('$out/bench.json')); print(d['ms_per_step'], {k: round(v,3) for k,v in d['config']['kernel_family_ms'].items()}, d['roofline']['frac'])" || tail -5 $out/bench.err
HODLR_ACA_NOGRAPH=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv python tools/prof_step.py cfg3 1 > /dev/null 2>&1
python tools/launch_summary.py $out/launches.csv

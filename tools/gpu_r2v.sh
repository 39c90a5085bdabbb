out=gpurun_out/r2v; mkdir -p $out
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $out/bench.json 2> $out/bench.err; tail -1 $out/bench.err | cut -c1-200
python -c "import json; d=json.load(open('$out/bench.json')); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['combined']['frac'], d['config']['kernel_family_ms'])"
HODLR_ACA_NOGRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launch.csv python tools/prof_step.py cfg3 1 > /dev/null 2>&1
python tools/launch_summary.py $out/launch.csv 2>/dev/null | head -4
timeout 3000 python -m pytest tests -m gpu -q -x 2>&1 | tail -4

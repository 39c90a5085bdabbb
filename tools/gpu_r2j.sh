out=gpurun_out/r2j; mkdir -p $out
HODLR_LIB=$PWD/paper_1403_6015_b200/libhodlr_trace.so timeout 300 python tools/prof_step.py cfg3 2 2>&1 | grep "tree d=" | tail -13
HODLR_LIB=$PWD/paper_1403_6015_b200/libhodlr_trace.so timeout 300 python tools/prof_step.py cfg1 2 2>&1 | grep "tree d=" | tail -5
timeout 300 python tools/e2e_probe.py 8
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $out/bench.json 2> $out/bench.err; tail -2 $out/bench.err
python -c "import json; d=json.load(open('$out/bench.json')); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['combined']['frac'], d['config']['kernel_family_ms'])"
HODLR_ACA_NOGRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launch.csv python tools/prof_step.py cfg3 1 > /dev/null 2>&1
python tools/launch_summary.py $out/launch.csv | head -8

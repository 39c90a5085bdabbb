out=gpurun_out/r2e; mkdir -p $out
timeout 300 python tools/e2e_probe.py 12
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $out/bench.json 2> $out/bench.err; tail -2 $out/bench.err
python -c "import json; d=json.load(open('$out/bench.json')); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['combined']['frac'], d['config']['kernel_family_ms'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launch.csv python tools/prof_step.py cfg3 1 > /dev/null 2>&1
python tools/launch_summary.py $out/launch.csv | head -12
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tree_factor --launch-skip 12 --launch-count 1 -o $out/tree_root python tools/prof_step.py cfg3 1 > /dev/null 2>&1
ncu -i $out/tree_root.ncu-rep --page source --csv --print-source sass > $out/tree_root_source.csv 2>/dev/null; ls -la $out

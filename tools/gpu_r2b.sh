set -x
out=gpurun_out/r2b; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_parity.py -x -q -k "not full_size and not extreme and not cfg4_sweep" 2>&1 | tail -15
timeout 300 python bench.py --steps 5 --warmup 3 > $out/bench.json 2> $out/bench.err; tail -3 $out/bench.err
python -c "import json; d=json.load(open('$out/bench.json')); print(d['ms_per_step'], d['e2e']['ms_per_step'], {k: round(v,3) for k,v in d['config']['kernel_family_ms'].items()}, d['roofline']['combined']['frac'], d['roofline']['frac'], d['cpu_baseline'])"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $out/traffic.csv python tools/prof_step.py cfg3 2 > /dev/null 2>&1
python tools/ncu_traffic.py $out/traffic.csv $out/traffic.json

out=gpurun_out/r2q; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -s -k "full_size_cfg5_vs_oracle_golden" 2>&1 | grep -E "cfg5|passed|failed|Error"
timeout 900 python tools/diag_fullsize.py cfg3 1048576 1e-12 2>&1 | grep -v "    block" | tail -6
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $out/bench.json 2> $out/bench.err; tail -1 $out/bench.err
python -c "import json; d=json.load(open('$out/bench.json')); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['combined']['frac'], d['config']['kernel_family_ms'])"
timeout 900 python tools/project_scaling.py cfg3 $out/scaling.json 2>&1 | tail -5
timeout 900 python tools/all_configs.py $out/configs.json 2>&1 | grep cfg4

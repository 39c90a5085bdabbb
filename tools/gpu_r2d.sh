set -x
out=gpurun_out/r2d; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_kernels.py -x -q -k "not full_size and not extreme" 2>&1 | tail -3
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $out/bench.json 2> $out/bench.err; tail -3 $out/bench.err
python -c "import json; d=json.load(open('$out/bench.json')); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['combined']['frac'], d['roofline']['frac']); [print(k['family'], round(k['ms'],3), k['bound'], round(k['frac'],3)) for k in d['roofline']['all_kernels']]"
HODLR_ACA_NOGRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $out/traffic.csv python tools/prof_step.py cfg3 2 > /dev/null 2>&1
python tools/ncu_traffic.py $out/traffic.csv $out/traffic.json
python tools/launch_summary.py $out/traffic.csv | head -30
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "full_size_cfg5_vs_oracle_golden or full_size_cfg3_parity" -s 2>&1 | grep -E "cfg5|cfg3|passed|failed|Error" | head

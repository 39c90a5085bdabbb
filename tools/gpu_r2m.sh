out=gpurun_out/r2m; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_predict.py tests/test_gpu_dist.py tests/test_gpu_apply.py tests/test_gpu_noise.py tests/test_gpu_kernels.py -x -q -k "not full_size and not extreme and not cfg4_sweep" 2>&1 | tail -4
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $out/bench.json 2> $out/bench.err; tail -2 $out/bench.err
python -c "import json; d=json.load(open('$out/bench.json')); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['combined']['frac'], d['config']['kernel_family_ms'])"
timeout 900 python tools/all_configs.py $out/configs.json 2>&1 | tail -1

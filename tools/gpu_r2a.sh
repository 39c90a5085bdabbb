set -x
mkdir -p gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "rank_cap_change or forced_ranks or config_parity or cfg4_sweep or edge or unsorted" 2>&1 | tail -15
timeout 900 python tools/diag_fullsize.py cfg3 1048576 1e-12 2>&1 | tail -30
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2a/bench.json 2> gpurun_out/r2a/bench.err; tail -3 gpurun_out/r2a/bench.err
python -c "import json; d=json.load(open('gpurun_out/r2a/bench.json')); print(d['ms_per_step'], d['e2e'], {k: round(v,3) for k,v in d['config']['kernel_family_ms'].items()})"

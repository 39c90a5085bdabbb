out=gpurun_out/r2o; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q -k "not full_size and not extreme and not cfg4_sweep" 2>&1 | tail -3
timeout 900 python tools/all_configs.py $out/configs.json 2>&1 | tail -1

out=gpurun_out/r2k; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_noise.py -x -q 2>&1 | tail -3
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > $out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 $out/sanitizer_$tool.log
done

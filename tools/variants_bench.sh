#!/bin/bash
# On the GPU box: bench each variant library (5 steps) and print step / family times.  bash tools/variants_bench.sh name ...
for name in base "$@"; do
  lib=""; [ "$name" != base ] && lib=paper_1403_6015_b200/var/libhodlr_$name.so
  HODLR_LIB=$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /tmp/vb.json 2>/tmp/vb.err
  python -c "import json; d=json.load(open('/tmp/vb.json')); print('$name', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['config']['kernel_family_ms'].items()})" 2>/dev/null \
    || { echo "$name FAILED:"; tail -4 /tmp/vb.err | sed 's/^/    | /'; }
done

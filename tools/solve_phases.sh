#!/bin/bash
# On the GPU box: solve leaf-up / leaf-down phase times (HODLR_TRACE stamps) per variant library.
for name in base "$@"; do
  lib=""; [ "$name" != base ] && lib=paper_1403_6015_b200/var/libhodlr_$name.so
  echo "$name $(HODLR_LIB=$lib HODLR_TRACE=1 timeout 120 python tools/prof_step.py cfg3 2 2>&1 | grep 'solve phases' | tail -1 | awk '{s=0; for(i=5;i<=NF;i++) s+=$i; print "leaf_up", $5, "leaf_down", $NF, "total", s}')"
done

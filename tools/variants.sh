#!/bin/bash
# Build library variants with -D overrides into paper_1403_6015_b200/var/ (they travel with gpurun), e.g.
#   bash tools/variants.sh "sub128:-DACA_SUB=128" "fused2k:-DACA_FUSED_MAX=2048"
# then on the GPU box: HODLR_LIB=paper_1403_6015_b200/var/libhodlr_<name>.so python bench.py ...
mkdir -p paper_1403_6015_b200/var
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    --expt-relaxed-constexpr $flags -o paper_1403_6015_b200/var/libhodlr_$name.so paper_1403_6015_b200/csrc/*.cu 2>&1 \
    | grep -E " error|error:" ; echo "built $name ($flags)"
done

#!/bin/bash
# Build experiment variants of the CUDA library into build/variants/<name>.so
# usage: bash tools/build_variants.sh name1:"-DFOO=1 -DBAR=0" name2:"..."
set -e
cd "$(dirname "$0")/.."
mkdir -p build/variants
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC -shared -cudart static $flags -o build/variants/$name.so \
    paper_2303_11767_b200/csrc/dgswe_b200.cu &
done
wait
ls -la build/variants

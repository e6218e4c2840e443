#!/bin/bash
# Build experiment variants of the CUDA library into build/variants/<name>.so
# (every degree unit, own object directory; variants build one after another)
# usage: bash tools/build_variants.sh name1:"-DFOO=1 -DBAR=0" name2:"..."
set -e
cd "$(dirname "$0")/.."
mkdir -p build/variants
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  python -c "
import sys; sys.path.insert(0, '.')
from paper_2303_11767_b200 import build
print(build.build(force=True, out='build/variants/$name.so', extra='$flags'.split()))"
done
ls -la build/variants/*.so

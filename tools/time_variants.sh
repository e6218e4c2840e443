#!/bin/bash
# kernel-only timing of every build/variants/*.so (twice, interleaved)
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for so in build/variants/*.so; do
    DGSWE_LIB=$PWD/$so timeout 300 python tools/time_stage.py "$@" 2>&1 | tail -1
  done
done

#!/bin/bash
# Time each build/variants/*.so with bench.py (kernel-only numbers), twice, interleaved.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
for so in build/variants/*.so; do
  n=$(basename $so .so)
  DGSWE_LIB=$PWD/$so timeout 300 python bench.py --steps ${STEPS:-100} --warmup 5 --no-cpu ${BENCH_ARGS:-} > gpurun_out/var_$n.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/var_$n.json')); r=d['roofline']
print('$n', round(r['frac'],4), {k: round(v*1e3,1) for k,v in r['per_stage_ms'].items()})"
done
done

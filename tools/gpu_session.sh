#!/bin/bash
# One gpurun session: tests, bench, ncu launch list and a full capture of the stage kernel.
# usage: bash tools/gpu_session.sh <tag> [tests|bench|ncu|all]...
set -u
TAG=${1:-r01}; shift
WHAT=${@:-all}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
for w in $WHAT; do
  if [[ $w == tests || $w == all ]]; then
    timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc $?"
    tail -3 gpurun_out/${TAG}_pytest_gpu.log
  fi
  if [[ $w == bench || $w == all ]]; then
    timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc $?"
    cat gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
  fi
  if [[ $w == ncu || $w == all ]]; then
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
      --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu > /dev/null 2>&1; echo "ncu launches rc $?"
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 9 -c 3 \
      -o gpurun_out/${TAG}_stage -f python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu full rc $?"
    tail -3 gpurun_out/${TAG}_ncu_full.log
  fi
done

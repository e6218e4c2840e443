set -u
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 300 python tools/time_stage.py 2>&1 | tail -1
timeout 300 python tools/time_stage.py 1440 720 3 2.5e-3 30 2>&1 | tail -1
DGSWE_LIB=$PWD/build/variants/timing.so timeout 300 python tools/phase_timing.py 2>&1 | tail -6
for c in c4 c2; do timeout 300 python bench.py --config $c --steps 50 --no-cpu > gpurun_out/n_$c.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/n_$c.json'));print('$c', d['value'], d['roofline']['frac'])"; done

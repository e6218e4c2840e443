"""bench.py's reference arm (the driver's `--impl reference` run) on CPU:
the JSON line contract, rank > 0 silence, and the warm-up floor."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CMD = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c2",
       "--steps", "1", "--warmup", "3", "--no-ref-python"]


def test_reference_arm_line():
    out = subprocess.run(CMD, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == "DOF-updates/sec (fp64, per RK stage)"
    assert line["value"] > 0 and line["unit"] == "DOF-updates/s" and line["higher_is_better"] is True
    assert line["steps"] == 1 and line["warmup"] == 3 and line["dtype"] == "f64"
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "DOF-updates/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["config"]["nx"] == 360 and line["config"]["p"] == 3


def test_reference_arm_other_ranks_silent():
    env = dict(os.environ, RANK="1")
    out = subprocess.run(CMD, capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_warmup_floor():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--warmup", "2"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode != 0 and "warmup" in (out.stderr + out.stdout)

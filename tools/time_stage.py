"""Kernel-only timing of K fused SSPRK3 steps (no status checks; for
experiment builds selected with DGSWE_LIB).  Prints us per stage and the
HBM roofline fraction at 21.33 B/DOF.

    DGSWE_LIB=build/variants/x.so python tools/time_stage.py [nx ny p dt K]
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2303_11767_b200 import SpatialOperator, build_case, default_config  # noqa: E402


def main():
    a = sys.argv[1:]
    nx, ny, p = (int(x) for x in (a[0:3] if len(a) >= 3 else (720, 360, 3)))
    dt = float(a[3]) if len(a) > 3 else 5e-3
    K = int(a[4]) if len(a) > 4 else 50
    cfg = default_config("williamson_tc6").override(nx=nx, ny=ny, p=p)
    setup = build_case(cfg)
    op = SpatialOperator(setup.mesh, p, setup.model)
    st = op.project_state(setup.ic, device=True)
    x0 = st.data.clone()
    best = 1e30
    for rep in range(3):
        st.data.copy_(x0)
        op.ssprk3_steps(st, dt, K)          # graph build + warm
        st.data.copy_(x0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        op.ssprk3_steps(st, dt, K)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / (3 * K) * 1e3)
    op.status(reset=True)
    dofs = nx * ny * 3 * (p + 1) ** 2
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6552.6)
    frac = dofs * (64.0 / 3.0) / (best * 1e-6) / 1e9 / peak
    tag = os.path.basename(os.environ.get("DGSWE_LIB", "in-tree"))
    print(f"{tag:20s} {best:8.2f} us/stage  frac {frac:.4f}")


if __name__ == "__main__":
    main()

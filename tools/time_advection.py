"""Kernel-only timing of the linear advection stage kernel (advection.py,
csrc/dgswe_adv.cuh): K fused SSPRK3 steps (AdvectionOperator.rk_steps) on
an nx x ny periodic grid of degree p, CUDA events around the steps.
Prints us per stage and the HBM roofline fraction at the stage's
algorithmic bytes (SSPRK3 Shu-Osher: 16 / 24 / 24 B per DOF, i.e. 64/3).

    python tools/time_advection.py [nx ny p K]
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2303_11767_b200 as P  # noqa: E402


def main():
    a = sys.argv[1:]
    nx, ny, p = (int(x) for x in (a[0:3] if len(a) >= 3 else (4096, 4096, 3)))
    K = int(a[3]) if len(a) > 3 else 20
    setup = P.build_case(P.default_config("advection_sine").override(nx=nx, ny=ny, p=p))
    op = P.AdvectionOperator(setup.mesh, p, setup.model)
    st = op.zero_state()
    st.data.normal_()
    dt = 0.1 / nx
    op.rk_steps(st, dt, 3, 3)                     # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    op.rk_steps(st, dt, K, 3)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / (3 * K) * 1e3
    dofs = nx * ny * (p + 1) ** 2
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6552.6)
    gbs = dofs * (64.0 / 3.0) / (us * 1e-6) / 1e9
    print(json.dumps({"kernel": f"dgswe::adv_stage_kernel<{p}>", "nx": nx, "ny": ny, "p": p, "dofs": dofs,
                      "us_per_stage": us, "dof_updates_per_s": dofs / (us * 1e-6), "achieved_gbs": gbs,
                      "peak_gbs": peak, "frac": gbs / peak}))


if __name__ == "__main__":
    main()

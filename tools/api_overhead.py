"""Per-step host overhead of the reference-API rk_step on the C3 grid:
rk_step(state, op.assemble_rhs, dt, tableau(3)) against the step's graph
replays alone (the GPU-bound floor).

    python tools/api_overhead.py
"""
import sys
import time
import os

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_11767_b200 as P  # noqa: E402
from paper_2303_11767_b200 import stepping  # noqa: E402


def main():
    setup = P.build_case(P.default_config("williamson_tc6").override(nx=720, ny=360, p=3))
    op = P.SpatialOperator(setup.mesh, 3, setup.model)
    st = op.project_state(setup.ic)
    tab = P.tableau(3)
    ws = stepping._RKWorkspace(st, tab.s)
    for _ in range(5):
        P.rk_step(st, op.assemble_rhs, 5e-3, tab, ws)
    torch.cuda.synchronize()
    n = 200
    t0 = time.perf_counter()
    for _ in range(n):
        P.rk_step(st, op.assemble_rhs, 5e-3, tab, ws)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    bufs = [ws.stage_input] + list(ws.k) + [ws.spare]
    for _ in range(3):
        op.rk_step_fused(st, 5e-3, 3, bufs)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    for _ in range(n):
        op.rk_step_fused(st, 5e-3, 3, bufs)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"rk_step {(t1 - t0) / n * 1e6:.1f} us/step; graph replays alone {(t3 - t2) / n * 1e6:.1f} us/step")


if __name__ == "__main__":
    main()

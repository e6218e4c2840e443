"""End-to-end SSPRK3 step of a pinned host state at C3 (ssprk3_step_host)
against the number of latitude chunks of its copy/compute pipeline.

    python tools/e2e_chunks.py
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_11767_b200 as P  # noqa: E402


def main():
    setup = P.build_case(P.default_config("williamson_tc6").override(nx=720, ny=360, p=3))
    op = P.SpatialOperator(setup.mesh, 3, setup.model)
    st = op.project_state(setup.ic)
    host = torch.empty(op.state_shape, dtype=torch.float64, pin_memory=True)
    host.copy_(st.data.cpu())
    for ch in (8, 12, 14, 16, 18, 20, 24):
        for _ in range(3):
            op.ssprk3_step_host(host, 5e-3, chunks=ch)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter()
            for _ in range(20):
                op.ssprk3_step_host(host, 5e-3, chunks=ch)
            torch.cuda.synchronize()
            best = min(best, (time.perf_counter() - t0) / 20 * 1e3)
        print(ch, round(best, 3), "ms/step")


if __name__ == "__main__":
    main()

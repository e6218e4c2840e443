"""Per-role phase timing of the stage kernel (DG_TIMING experiment build).

    DGSWE_LIB=build/variants/<timing>.so python tools/phase_timing.py [nx ny p]
Prints average cycles per row for each warp role and phase.
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2303_11767_b200 import SpatialOperator, _lib, build_case, default_config  # noqa: E402


def main():
    a = sys.argv[1:]
    nx, ny, p = (int(x) for x in (a[0:3] if len(a) >= 3 else (720, 360, 3)))
    dt = 5e-3
    cfg = default_config("williamson_tc6").override(nx=nx, ny=ny, p=p)
    setup = build_case(cfg)
    op = SpatialOperator(setup.mesh, p, setup.model)
    st = op.project_state(setup.ic)
    lib = _lib.load()
    fn = getattr(lib, f"dgswe_debug_timing_p{p}")
    fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
    buf = (ctypes.c_ulonglong * 28)()
    op.ssprk3_steps(st, dt, 3)
    fn(buf)
    op.ssprk3_steps(st, dt, 20)
    torch.cuda.synchronize()
    fn(buf)
    a = np.array(list(buf), dtype=np.float64).reshape(4, 7)
    names = ["h", "hu", "hv", "face"]
    print("cycles/row  eval  ringwait  bar1  B-work  bar2  C-work  total   (face: -, -, bar1, yface, bar2, border)")
    for r in range(4):
        rows = a[r, 6]
        x = a[r, :6] / max(rows, 1)
        print(f"{names[r]:5s} " + " ".join(f"{y:7.0f}" for y in x) + f" {x.sum():8.0f}")


if __name__ == "__main__":
    main()

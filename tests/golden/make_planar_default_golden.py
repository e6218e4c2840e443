"""The reference's default f-plane run (cases.default_config("geostrophic_adjustment"):
50x50, p = 3, RK4, dt = 100 s, t_final = 36000 s: 360 steps) through the
UNMODIFIED reference's own ``integrate``; writes tests/golden/planar_default.npz
(final interior coefficients (3, nx, ny, nz, nphi), mass at t = 0 and at
t_final, the step count).  Run once in the build container:

    python tests/golden/make_planar_default_golden.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_dgswe")
sys.path.insert(0, REF)

from dgswe import cases, dg, diagnostics, timestep  # noqa: E402


def main():
    cfg = cases.default_config("geostrophic_adjustment")
    setup = cases.build_case(cfg)
    op = dg.SpatialOperator(setup.mesh, cfg.p, setup.model)
    st = op.project_state(setup.ic)
    m0 = diagnostics.mass_integral(st, op)
    ctl = timestep.TimeControls(t_final=cfg.t_final, dt=cfg.dt)
    st, log = timestep.integrate(st, op, ctl, timestep.tableau(cfg.rk))
    xT = np.stack([np.ascontiguousarray(st.interior_coeffs(n)) for n in st.names])
    np.savez_compressed(os.path.join(HERE, "planar_default.npz"), xT=xT,
                        mass=np.array([m0, diagnostics.mass_integral(st, op)]),
                        steps=np.array([log.steps]))
    print("steps", log.steps, "mass", m0)


if __name__ == "__main__":
    main()

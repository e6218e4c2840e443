"""The reference's default Williamson TC6 configuration
(cases.default_config("williamson_tc6"): 40x20, p = 3, RK4, dt = 4 s)
through the UNMODIFIED reference's own ``integrate`` for its first hour
(t_final = 3600 s, 900 steps; the configured 8 days would take the CPU
reference hours).  Writes tests/golden/tc6_default_1h.npz: final
coefficients, mass at 0 and 1 h, the step count.

    python tests/golden/make_tc6_default_golden.py
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

T_FINAL = 3600.0


def main():
    cfg = cases.default_config("williamson_tc6")
    setup = cases.build_case(cfg)
    op = dg.SpatialOperator(setup.mesh, cfg.p, setup.model)
    st = op.project_state(setup.ic)
    m0 = diagnostics.mass_integral(st, op)
    st, log = timestep.integrate(st, op, timestep.TimeControls(t_final=T_FINAL, dt=cfg.dt),
                                 timestep.tableau(cfg.rk))
    xT = np.stack([np.ascontiguousarray(st.interior_coeffs(n)) for n in st.names])
    np.savez_compressed(os.path.join(HERE, "tc6_default_1h.npz"), xT=xT,
                        mass=np.array([m0, diagnostics.mass_integral(st, op)]), steps=np.array([log.steps]))
    print("steps", log.steps)


if __name__ == "__main__":
    main()

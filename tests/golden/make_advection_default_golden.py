"""The reference's default advection run (cases.default_config("advection_sine"):
20x20, p = 2, RK4, Courant 0.2, t_final = 1: one full period) through the
UNMODIFIED reference's own ``integrate``; writes
tests/golden/advection_default.npz (final coefficients, the L2 error
against the exact solution, absolute and relative, the step count and dt).

    python tests/golden/make_advection_default_golden.py
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
    cfg = cases.default_config("advection_sine")
    setup = cases.build_case(cfg)
    op = dg.SpatialOperator(setup.mesh, cfg.p, setup.model)
    st = op.project_state(setup.ic)
    ctl = timestep.TimeControls(t_final=cfg.t_final, courant=cfg.courant)
    st, log = timestep.integrate(st, op, ctl, timestep.tableau(cfg.rk))
    xT = np.stack([np.ascontiguousarray(st.interior_coeffs(n)) for n in st.names])
    ex = setup.exact(cfg.t_final)
    np.savez_compressed(os.path.join(HERE, "advection_default.npz"), xT=xT,
                        err=np.array([diagnostics.l2_error(st, ex, op),
                                      diagnostics.l2_error(st, ex, op, relative=True)]),
                        steps=np.array([log.steps]), dt=np.array([log.dt]))
    print("steps", log.steps, "dt", log.dt)


if __name__ == "__main__":
    main()

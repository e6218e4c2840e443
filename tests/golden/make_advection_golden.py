"""Generate the linear-advection golden fixtures from the UNMODIFIED
reference package.

Run once in the build container (the only place /root/reference exists):

    python tests/golden/make_advection_golden.py

It imports ``dgswe`` from /root/reference/pkg/src read-only and writes
``tests/golden/advection.npz``: for each case (``advection_sine`` with the
mesh and degree overridden) the projected initial coefficients, the
right-hand side there, the state after N reference ``rk_step`` steps of
the case's tableau and its right-hand side, and the reference ``integrate``
result at a short final time with its L2 error against the exact
(translated) solution.  Arrays are (1, nx, ny, nz, nphi) interior
coefficients.  Nothing here is imported by the product.
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

# name, nx, ny, p, rk, dt, nsteps  (nx = 33 / 40: partial strips of 32 lanes)
CASES = [
    ("sine_20x20_p2", 20, 20, 2, 4, 0.005, 6),
    ("sine_33x10_p1", 33, 10, 1, 3, 0.01, 6),
    ("sine_16x12_p3", 16, 12, 3, 4, 0.002, 6),
    ("sine_12x8_p4", 12, 8, 4, 3, 0.002, 6),
    ("sine_40x7_p0", 40, 7, 0, 2, 0.005, 6),
    ("sine_10x9_p5", 10, 9, 5, 4, 0.001, 4),
]
T_FINAL = 0.05


def coeffs_of(st):
    return np.stack([np.ascontiguousarray(st.interior_coeffs(n)) for n in st.names])


def main():
    out = {}
    for name, nx, ny, p, rk, dt, nsteps in CASES:
        cfg = cases.default_config("advection_sine").override(nx=nx, ny=ny, p=p, rk=rk)
        setup = cases.build_case(cfg)
        op = dg.SpatialOperator(setup.mesh, p, setup.model)
        st = op.project_state(setup.ic)
        out[f"{name}/x0"] = coeffs_of(st)
        out[f"{name}/rhs0"] = coeffs_of(op.assemble_rhs(st))
        tab = timestep.tableau(rk)
        ws = timestep._RKWorkspace(st, tab.s)
        for _ in range(nsteps):
            timestep.rk_step(st, op.assemble_rhs, dt, tab, ws)
        out[f"{name}/xn"] = coeffs_of(st)
        out[f"{name}/rhsn"] = coeffs_of(op.assemble_rhs(st))
        # integrate to a short final time with the case's Courant control
        st2 = op.project_state(setup.ic)
        ctl = timestep.TimeControls(t_final=T_FINAL, courant=cfg.courant)
        st2, log = timestep.integrate(st2, op, ctl, tab)
        out[f"{name}/xT"] = coeffs_of(st2)
        out[f"{name}/errT"] = np.array([diagnostics.l2_error(st2, setup.exact(T_FINAL), op),
                                        diagnostics.l2_error(st2, setup.exact(T_FINAL), op, relative=True)])
        out[f"{name}/meta"] = np.array([nx, ny, p, rk, dt, nsteps, log.steps, log.dt])
        print(name, "done", flush=True)
    # a pinned global Rusanov alpha (dg.py:389-392) on the first case: RHS of
    # the N-step state and 3 more steps
    name, nx, ny, p, rk, dt, nsteps = CASES[0]
    cfg = cases.default_config("advection_sine").override(nx=nx, ny=ny, p=p, rk=rk)
    setup = cases.build_case(cfg)
    op = dg.SpatialOperator(setup.mesh, p, setup.model, rusanov=dg.RusanovParams("global", 2.5))
    st = op.zero_state()
    st.fields["u"].data[1:-1, 1:-1] = out[f"{name}/xn"][0]
    out[f"{name}/pinned/rhs"] = coeffs_of(op.assemble_rhs(st))
    tab = timestep.tableau(rk)
    ws = timestep._RKWorkspace(st, tab.s)
    for _ in range(3):
        timestep.rk_step(st, op.assemble_rhs, dt, tab, ws)
    out[f"{name}/pinned/x3"] = coeffs_of(st)
    np.savez_compressed(os.path.join(HERE, "advection.npz"), **out)


if __name__ == "__main__":
    main()

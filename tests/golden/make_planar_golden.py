"""Generate the planar (f-plane geostrophic adjustment) golden fixtures from
the UNMODIFIED reference package.

Run once in the build container (the only place /root/reference exists):

    python tests/golden/make_planar_golden.py

It imports ``dgswe`` from /root/reference/pkg/src read-only and writes
``tests/golden/planar.npz``: for each case the projected initial
coefficients, the right-hand side there, the state after N reference
``rk_step(tableau(3))`` steps (momentum non-zero by then) and the
right-hand side of that state, and the right-hand sides of both states
scaled by (1 + 2^-52) (the reference's own rounding sensitivity); for the
first case also the RHS and 3 more steps from the N-step state with the
global and a pinned Rusanov alpha.  Arrays
are (3, nx, ny, nz, nphi) interior
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

from dgswe import cases, dg, timestep  # noqa: E402

# name, nx, ny, p, dt, nsteps  (nx = 33: a partial second strip of 32 lanes)
CASES = [
    ("adj_16x12_p3", 16, 12, 3, 400.0, 5),
    ("adj_33x10_p1", 33, 10, 1, 800.0, 5),
    ("adj_24x8_p2", 24, 8, 2, 600.0, 5),
    ("adj_20x6_p4", 20, 6, 4, 300.0, 5),
]


def coeffs_of(st):
    return np.stack([np.ascontiguousarray(st.interior_coeffs(n)) for n in st.names])


def main():
    out = {}
    for name, nx, ny, p, dt, nsteps in CASES:
        cfg = cases.default_config("geostrophic_adjustment").override(nx=nx, ny=ny, p=p)
        setup = cases.build_case(cfg)
        op = dg.SpatialOperator(setup.mesh, p, setup.model)
        st = op.project_state(setup.ic)
        out[f"{name}/x0"] = coeffs_of(st)
        out[f"{name}/rhs0"] = coeffs_of(op.assemble_rhs(st))
        tab = timestep.tableau(3)
        ws = timestep._RKWorkspace(st, tab.s)
        for _ in range(nsteps):
            timestep.rk_step(st, op.assemble_rhs, dt, tab, ws)
        out[f"{name}/xn"] = coeffs_of(st)
        out[f"{name}/rhsn"] = coeffs_of(op.assemble_rhs(st))
        # the reference's own 1-ulp sensitivity: the RHS of the states scaled
        # by (1 + 2^-52) (the RHS is a cancellation of O(g h^2) pressure terms;
        # the GPU gate is a multiple of this spread)
        for tag, X in (("0", out[f"{name}/x0"]), ("n", out[f"{name}/xn"])):
            sp = op.zero_state()
            for v, nm in enumerate(sp.names):
                sp.fields[nm].data[1:-1, 1:-1] = X[v] * (1.0 + 2.0 ** -52)
            out[f"{name}/rhs{tag}_ulp"] = coeffs_of(op.assemble_rhs(sp))
        out[f"{name}/meta"] = np.array([nx, ny, p, dt, nsteps])
        print(name, "done", flush=True)
    # global Rusanov alpha (dg.py:385-421, mode "global") and a pinned one,
    # on the state after N steps of the first case: RHS and 3 further steps
    name, nx, ny, p, dt, nsteps = CASES[0]
    for tag, rus in (("global", dg.RusanovParams("global")), ("pinned", dg.RusanovParams("global", 250.0))):
        cfg = cases.default_config("geostrophic_adjustment").override(nx=nx, ny=ny, p=p)
        setup = cases.build_case(cfg)
        op = dg.SpatialOperator(setup.mesh, p, setup.model, rusanov=rus)
        st = op.zero_state()
        for v, nm in enumerate(st.names):
            st.fields[nm].data[1:-1, 1:-1] = out[f"{name}/xn"][v]
        out[f"{name}/{tag}/rhs"] = coeffs_of(op.assemble_rhs(st))
        tab = timestep.tableau(3)
        ws = timestep._RKWorkspace(st, tab.s)
        for _ in range(3):
            timestep.rk_step(st, op.assemble_rhs, dt, tab, ws)
        out[f"{name}/{tag}/x3"] = coeffs_of(st)
        # the reference's own 1-ulp sensitivity of those 3 steps (the gate's scale)
        st = op.zero_state()
        for v, nm in enumerate(st.names):
            st.fields[nm].data[1:-1, 1:-1] = out[f"{name}/xn"][v] * (1.0 + 2.0 ** -52)
        ws = timestep._RKWorkspace(st, tab.s)
        for _ in range(3):
            timestep.rk_step(st, op.assemble_rhs, dt, tab, ws)
        out[f"{name}/{tag}/x3_ulp"] = coeffs_of(st)
        print(name, tag, "done", flush=True)
    np.savez_compressed(os.path.join(HERE, "planar.npz"), **out)


if __name__ == "__main__":
    main()

"""The reference's default Williamson TC2 configuration
(cases.default_config("williamson_tc2"): 20x20, p = 3, RK4, Courant 0.2,
dt = 99.4 s) is unstable: the UNMODIFIED reference's ``integrate`` raises
DivergenceError (from a PositivityError inside the RHS) at step 7.  This
records the step, the time and the state the reference leaves behind
(u after step 6), and that state from a 1-ulp-perturbed start (the run is
chaotic by then), in tests/golden/tc2_default_failure.npz.

    python tests/golden/make_tc2_default_golden.py
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


def main():
    cfg = cases.default_config("williamson_tc2")
    setup = cases.build_case(cfg)
    op = dg.SpatialOperator(setup.mesh, cfg.p, setup.model)
    st = op.project_state(setup.ic)
    ctl = timestep.TimeControls(t_final=cfg.t_final, courant=cfg.courant)
    try:
        timestep.integrate(st, op, ctl, timestep.tableau(cfg.rk))
        raise SystemExit("the reference did not fail")
    except timestep.DivergenceError as e:
        step, t = e.step, e.t
    x = np.stack([np.ascontiguousarray(st.interior_coeffs(n)) for n in st.names])
    # the run is far past its stability limit, so rounding grows ~100x per
    # step: the reference's own spread under a 1-ulp change of the initial
    # state scales the state gate
    st = op.project_state(setup.ic)
    for n in st.names:
        st.fields[n].data[1:-1, 1:-1] *= 1.0 + 2.0 ** -52
    try:
        timestep.integrate(st, op, ctl, timestep.tableau(cfg.rk))
    except timestep.DivergenceError:
        pass
    x_ulp = np.stack([np.ascontiguousarray(st.interior_coeffs(n)) for n in st.names])
    np.savez_compressed(os.path.join(HERE, "tc2_default_failure.npz"), x=x, x_ulp=x_ulp,
                        step=np.array([step]), t=np.array([t]))
    print("step", step, "t", t)


if __name__ == "__main__":
    main()

"""GPU parity of the linear advection case (advection_sine on the doubly
periodic unit square, cases.py:99-110) against the unmodified reference's
own outputs (tests/golden/advection.npz, tests/golden/make_advection_golden.py).

The operator is linear, so the reference's 1-ulp sensitivity is the
rounding of the state itself: the RHS gate is 1e-13 of the RHS norm (the
nodal form and the reference's modal quadrature round differently); N
Butcher-form rk_step steps and integrate() to t = 0.05 within 1e-12
relative (the north star's 1e-11 gate with margin); the L2 error against
the translated exact solution within 1e-9 relative (+1e-13 absolute) of
the reference's.
"""

import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "advection.npz")
NAMES = ["sine_20x20_p2", "sine_33x10_p1", "sine_16x12_p3", "sine_12x8_p4", "sine_40x7_p0", "sine_10x9_p5"]
T_FINAL = 0.05


@pytest.fixture(scope="module")
def P():
    import paper_2303_11767_b200 as P
    torch.cuda.set_device(0)
    return P


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLDEN)


def make(P, gold, name, nz=1):
    nx, ny, p, rk, dt, nsteps, n_int, dt_int = gold[f"{name}/meta"]
    cfg = P.default_config("advection_sine").override(nx=int(nx), ny=int(ny), p=int(p), rk=int(rk))
    setup = P.build_case(cfg)
    op = P.AdvectionOperator(setup.mesh, int(p), setup.model, nz=nz)
    return setup, op, cfg, float(dt), int(nsteps)


def rel(got, ref):
    return np.linalg.norm(got - ref) / np.linalg.norm(ref)


@pytest.mark.parametrize("name", NAMES)
def test_advection_rhs_vs_reference(P, gold, name):
    setup, op, cfg, dt, nsteps = make(P, gold, name)
    st = op.project_state(setup.ic)
    assert np.array_equal(st.to_numpy(), gold[f"{name}/x0"])          # host projection: the reference's bits
    assert rel(op.assemble_rhs(st).to_numpy(), gold[f"{name}/rhs0"]) <= 1e-13
    xn = op.state_from_coeffs({"u": gold[f"{name}/xn"][0][:, :, 0, :]})
    assert rel(op.assemble_rhs(xn).to_numpy(), gold[f"{name}/rhsn"]) <= 1e-13


@pytest.mark.parametrize("name", NAMES)
def test_advection_steps_vs_reference(P, gold, name):
    setup, op, cfg, dt, nsteps = make(P, gold, name)
    st = op.project_state(setup.ic)
    tab = P.tableau(cfg.rk)
    ws = P.stepping._RKWorkspace(st, tab.s)
    for _ in range(nsteps):
        P.rk_step(st, op.assemble_rhs, dt, tab, ws)
    assert rel(st.to_numpy(), gold[f"{name}/xn"]) <= 1e-12


@pytest.mark.parametrize("name", NAMES)
def test_advection_integrate_vs_reference(P, gold, name):
    setup, op, cfg, dt, nsteps = make(P, gold, name)
    st = op.project_state(setup.ic)
    m0 = P.mass_integral(st, op)
    ctl = P.TimeControls(t_final=T_FINAL, courant=cfg.courant)
    st, log = P.integrate(st, op, ctl, P.tableau(cfg.rk))
    meta = gold[f"{name}/meta"]
    assert log.steps == int(meta[6]) and log.dt == meta[7]
    assert rel(st.to_numpy(), gold[f"{name}/xT"]) <= 1e-12
    err, err_rel = gold[f"{name}/errT"]
    # the state agrees to ~1e-13 of its O(1) norm, which bounds the error's difference
    assert abs(P.l2_error(st, setup.exact(T_FINAL), op) - err) <= 1e-9 * err + 1e-13
    assert abs(P.l2_error(st, setup.exact(T_FINAL), op, relative=True) - err_rel) <= 1e-9 * err_rel + 1e-13
    # the mean of sin(2 pi x) sin(2 pi y) is zero; the scheme conserves it
    assert abs(P.mass_integral(st, op) - m0) <= 1e-14


def test_advection_layers_and_stage_form(P, gold):
    """nz layers are independent copies; Y = a U + b X + g RHS(X) matches the
    composition of its parts; U may alias Y (the in-place last stage)."""
    name = "sine_16x12_p3"
    setup, op, cfg, dt, nsteps = make(P, gold, name, nz=3)
    st = op.project_state(setup.ic)
    st.data[1] *= -2.0
    st.data[2] *= 0.5
    r = op.assemble_rhs(st).data
    assert torch.equal(r[1], r[0] * -2.0) and torch.equal(r[2], r[0] * 0.5)     # power-of-2 scalings are exact
    U = op.state_from_coeffs({"u": gold[f"{name}/xn"][0][:, :, 0, :]})
    Y = op.zero_state()
    op.stage(0.25, U, 0.75, st, 0.125, Y)
    want = (U.data * 0.25 + (st.data * 0.75 + r * 0.125))
    assert torch.allclose(Y.data, want, rtol=1e-14, atol=1e-15 * float(want.abs().max()))
    Z = U.copy()
    op.stage(0.25, Z, 0.75, st, 0.125, Z)
    assert torch.equal(Z.data, Y.data)
    with pytest.raises(RuntimeError):
        op.stage(0.0, None, 1.0, st, 1.0, st)                          # X aliasing Y is rejected


@pytest.mark.parametrize("order", [1, 2, 3])
def test_advection_fused_steps(P, gold, order):
    """Shu-Osher stage form vs the Butcher-form rk_step of the same tableau
    (the two orderings round differently: 1e-13 relative)."""
    name = "sine_20x20_p2"
    setup, op, cfg, dt, nsteps = make(P, gold, name)
    a = op.project_state(setup.ic)
    b = op.project_state(setup.ic)
    op.rk_steps(a, dt, 10, order)
    tab = P.tableau(order)
    ws = P.stepping._RKWorkspace(b, tab.s)
    for _ in range(10):
        P.rk_step(b, op.assemble_rhs, dt, tab, ws)
    assert rel(a.to_numpy(), b.to_numpy()) <= 1e-13


def test_advection_convergence(P):
    """Order p+1 of the L2 error at t = 0.05 (SSPRK3, small dt): the
    reference's convergence study for this case (cases.py:99-110)."""
    errs = []
    for nx in (8, 16):
        setup = P.build_case(P.default_config("advection_sine").override(nx=nx, ny=nx, p=2, rk=3))
        op = P.AdvectionOperator(setup.mesh, 2, setup.model)
        st = op.project_state(setup.ic)
        op.rk_steps(st, 0.05 / 200, 200, 3)
        errs.append(P.l2_error(st, setup.exact(0.05), op))
    rate = P.convergence_rate(errs[0], 1.0 / 8, errs[1], 1.0 / 16)
    assert rate > 2.7, (errs, rate)


def test_advection_pinned_alpha_vs_reference(P, gold):
    """RusanovParams("global", 2.5) (dg.py:389-392): one RHS and 3 steps."""
    name = "sine_20x20_p2"
    nx, ny, p, rk, dt, nsteps, n_int, dt_int = gold[f"{name}/meta"]
    setup = P.build_case(P.default_config("advection_sine").override(nx=int(nx), ny=int(ny), p=int(p), rk=int(rk)))
    op = P.AdvectionOperator(setup.mesh, int(p), setup.model, rusanov=P.RusanovParams("global", 2.5))
    x = op.state_from_coeffs({"u": gold[f"{name}/xn"][0][:, :, 0, :]})
    assert rel(op.assemble_rhs(x).to_numpy(), gold[f"{name}/pinned/rhs"]) <= 1e-13
    tab = P.tableau(int(rk))
    ws = P.stepping._RKWorkspace(x, tab.s)
    for _ in range(3):
        P.rk_step(x, op.assemble_rhs, float(dt), tab, ws)
    assert rel(x.to_numpy(), gold[f"{name}/pinned/x3"]) <= 1e-12
    default = P.AdvectionOperator(setup.mesh, int(p), setup.model, rusanov=P.RusanovParams("global"))
    assert rel(default.assemble_rhs(x).to_numpy(), P.AdvectionOperator(setup.mesh, int(p), setup.model)
               .assemble_rhs(x).to_numpy()) == 0.0           # global == local for constant beta


def test_advection_default_run_vs_reference(P):
    """The reference's default advection run (20x20, p = 2, RK4, Courant
    0.2, one period) through integrate(): final state within 1e-12 relative
    of the reference's own run, its L2 error against the exact solution
    within 1e-9 relative (tests/golden/advection_default.npz)."""
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "advection_default.npz"))
    cfg = P.default_config("advection_sine")
    setup = P.build_case(cfg)
    op = P.AdvectionOperator(setup.mesh, cfg.p, setup.model)
    st = op.project_state(setup.ic)
    st, log = P.integrate(st, op, P.TimeControls(t_final=cfg.t_final, courant=cfg.courant), P.tableau(cfg.rk))
    assert log.steps == int(g["steps"][0]) and log.dt == float(g["dt"][0])
    assert rel(st.to_numpy(), g["xT"]) <= 1e-12
    err, err_rel = g["err"]
    assert abs(P.l2_error(st, setup.exact(cfg.t_final), op) - err) <= 1e-9 * err
    assert abs(P.l2_error(st, setup.exact(cfg.t_final), op, relative=True) - err_rel) <= 1e-9 * err_rel


def test_advection_op_recorder(P, gold):
    """set_op_recorder (fields.py:66-76) sees one record per advection launch,
    with the one-variable DOF count."""
    name = "sine_16x12_p3"
    setup, op, cfg, dt, nsteps = make(P, gold, name)
    st = op.project_state(setup.ic)
    seen = []

    class Rec:
        def record(self, kind, opname, rgn, flops, nbytes):
            seen.append((kind, opname, rgn.dofs, nbytes))

    P.set_op_recorder(Rec())
    try:
        op.rk_steps(st, dt, 2, 3)
    finally:
        P.set_op_recorder(None)
    dofs = 16 * 12 * 16
    assert len(seen) == 6 and all(s[1] == "dgswe_adv_stage" and s[2] == dofs for s in seen)
    assert [s[3] for s in seen[:3]] == [16 * dofs, 24 * dofs, 24 * dofs]

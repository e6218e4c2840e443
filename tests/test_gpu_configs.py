"""GPU parity at BASELINE.json's configurations, at full size.

The oracle (bit-exact C restatement of the reference, OpenMP) runs the same
steps on the host; its result is itself pinned to the reference by the
SHA-256 fixtures make_golden.py generated from the unmodified reference at
these sizes (cases c2_full / c3_full / c4_full), so every comparison below
is transitively against the reference.

Gates (north star: rel L2 <= 1e-11 after N steps, mass drift matching to
1e-13), plus two that stay sharp when the state barely moves (tiny dt):
* one RHS through the reference's entry point (assemble_rhs: the modal
  single-launch kernel) within 20x the oracle's own 1-ulp sensitivity;
* the state error relative to the state CHANGE over the run,
  ||U_gpu - U_orc|| / ||U_orc - U_0|| <= 1e-6: an RHS error of relative size
  e shows up here as ~e, independent of dt (measured 1.6e-7 - 2e-7 at C4 /
  TC5 for 3 steps of 5e-4 s: the per-step rounding of the update, ~eps ||U||,
  against a per-step change of ~1e-8 ||U||; not for TC2, a steady state
  whose change is itself discretisation error);
* TC2 (C2): the analytic L2 error of h (diagnostics.l2_error) within 1e-11
  of the reference's value (|l2(a) - l2(b)| <= ||a - b|| / ||h_exact||, so
  this is implied by, and as tight as, the state gate).
"""

import hashlib

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2303_11767_b200 as P
    torch.cuda.set_device(0)
    return P


def sha16(X):
    h = hashlib.sha256()
    for v in range(X.shape[0]):
        h.update(np.ascontiguousarray(X[v]).tobytes())
    return h.hexdigest()[:16]


def rel(a, b, v):
    return float(np.linalg.norm(a[v] - b[v]) / max(np.linalg.norm(b[v]), 1e-300))


def gate_states(got, ref, X0, case, tol=1e-11, tol_change=1e-6):
    assert np.all(np.isfinite(got))
    assert rel(got, ref, 0) <= tol, ("h", rel(got, ref, 0))
    assert rel(got, ref, 1) <= tol, ("hu", rel(got, ref, 1))
    mom = np.sqrt(np.linalg.norm(ref[1]) ** 2 + np.linalg.norm(ref[2]) ** 2)
    assert np.linalg.norm(got[2] - ref[2]) / mom <= tol
    if case == "williamson_tc6":      # TC2 / TC5 hv: discretisation-error sized
        assert rel(got, ref, 2) <= tol, ("hv", rel(got, ref, 2))
    if tol_change is None:
        return None
    change = np.linalg.norm(ref - X0)
    assert change > 0
    err = np.linalg.norm(got - ref) / change
    assert err <= tol_change, ("error / state change", err)
    return err


def rhs_gate(orc, X, K):
    Kr = orc.rhs(X)
    rng = np.random.default_rng(0)
    Kp = orc.rhs(X * (1.0 + rng.integers(-1, 2, size=X.shape) * 2.0 ** -52))
    for v in range(3):
        sens = float(np.linalg.norm(Kp[v] - Kr[v]) / np.linalg.norm(Kr[v]))
        assert rel(K, Kr, v) <= max(20 * sens, 1e-13), (v, rel(K, Kr, v), sens)


def test_c2_config(P, golden, oracle_mod):
    """C2: TC2, p=3, 360x180, dt=0.05 s, 100 SSPRK3 steps through
    integrate() (fused CUDA-graph batches) vs 100 Butcher steps of the
    oracle (== the reference: sha_final); analytic L2 and mass vs the
    reference's own values."""
    meta, _ = golden
    e = meta["cases"]["c2_full"]
    t, orc, X = oracle_mod.build_case("williamson_tc2", 360, 180, 3)
    assert sha16(X) == e["sha_ic"]
    cfg = P.default_config("williamson_tc2").override(nx=360, ny=180, p=3)
    setup = P.build_case(cfg)
    op = P.SpatialOperator(setup.mesh, 3, setup.model)
    st = op.project_state(setup.ic)
    assert np.array_equal(st.to_numpy(), X)
    rhs_gate(orc, X, op.assemble_rhs(st).to_numpy())
    U, status, _ = orc.rk_steps(X, e["dt"], 3, e["nsteps"])
    assert status == 0 and sha16(U) == e["sha_final"]
    st, log = P.integrate(st, op, P.TimeControls(e["dt"] * e["nsteps"], dt=e["dt"]), P.tableau(3))
    assert log.steps == e["nsteps"]
    got = st.to_numpy()
    # TC2 is steady: its state change is itself discretisation error (~1e-11
    # relative), so the change-normalised gate does not apply (measured 7e-5:
    # 1e-15 relative rounding); the RHS gate above is the sharp one
    gate_states(got, U, X, "williamson_tc2", tol_change=None)
    l2 = P.l2_error(st, setup.exact(e["dt"] * e["nsteps"]), op, "h", relative=True)
    assert abs(l2 - e["l2_h_rel_final"]) <= 1e-11, (l2, e["l2_h_rel_final"])
    m0, m1 = e["mass_ic"][0], e["mass_final"][0]
    mg0 = P.mass_integral_host(op.state_from_array(X), op)
    mg1 = P.mass_integral_host(st, op)
    assert abs((mg1 - mg0) - (m1 - m0)) <= 1e-13 * abs(m0)


@pytest.mark.parametrize("path", ["rk_steps", "rk_step"])
def test_c3_config(P, golden, oracle_mod, path):
    """C3 (the benchmarked workload): TC6, p=3, 720x360, dt=5e-3 s, 20
    steps -- through the fused nodal stages of the bench (rk_steps) and
    through the reference's own rk_step(state, op.assemble_rhs, dt,
    tableau(3)) (modal single-launch stages) -- vs the oracle's Butcher
    steps (== the reference: sha_final)."""
    meta, _ = golden
    e = meta["cases"]["c3_full"]
    t, orc, X = oracle_mod.build_case("williamson_tc6", 720, 360, 3)
    assert sha16(X) == e["sha_ic"]
    setup = P.build_case(P.default_config("williamson_tc6").override(nx=720, ny=360, p=3))
    op = P.SpatialOperator(setup.mesh, 3, setup.model)
    st = op.state_from_array(X)
    if path == "rk_steps":
        rhs_gate(orc, X, op.assemble_rhs(st).to_numpy())
    U, status, _ = orc.rk_steps(X, e["dt"], 3, e["nsteps"])
    assert status == 0 and sha16(U) == e["sha_final"]
    if path == "rk_steps":
        op.ssprk3_steps(st, e["dt"], e["nsteps"])
        assert op.status()[0] == 0
    else:
        tab = P.tableau(3)
        ws = P.stepping._RKWorkspace(st, tab.s)
        for _ in range(e["nsteps"]):
            P.rk_step(st, op.assemble_rhs, e["dt"], tab, ws)
    gate_states(st.to_numpy(), U, X, "williamson_tc6")
    m0 = P.mass_integral_host(op.state_from_array(X), op)
    drift = P.mass_integral_host(st, op) - m0
    assert abs(drift - (e["mass_final"][0] - e["mass_ic"][0])) <= 1e-13 * abs(m0)


def test_c4_config(P, golden, oracle_mod):
    """C4 shape: p=4, 1440x720, TC6 IC, dt=5e-4 s, 3 steps vs the oracle
    (== the reference: sha_final), device IC projection vs the host one."""
    meta, _ = golden
    e = meta["cases"]["c4_full"]
    t, orc, X = oracle_mod.build_case("williamson_tc6", 1440, 720, 4)
    assert sha16(X) == e["sha_ic"]
    setup = P.build_case(P.default_config("williamson_tc6").override(nx=1440, ny=720, p=4))
    op = P.SpatialOperator(setup.mesh, 4, setup.model)
    sd = op.project_state(setup.ic, device=True).to_numpy()
    for v in range(3):
        assert np.linalg.norm(sd[v] - X[v]) <= 1e-13 * max(np.linalg.norm(X[v]), np.linalg.norm(X[0]))
    st = op.state_from_array(X)
    rhs_gate(orc, X, op.assemble_rhs(st).to_numpy())
    U, status, _ = orc.rk_steps(X, e["dt"], 3, e["nsteps"])
    assert status == 0 and sha16(U) == e["sha_final"]
    op.ssprk3_steps(st, e["dt"], e["nsteps"])
    assert op.status()[0] == 0
    gate_states(st.to_numpy(), U, X, "williamson_tc6")
    m0 = P.mass_integral(op.state_from_array(X), op)
    drift = P.mass_integral(st, op) - m0
    assert abs(drift - (e["mass_final"][0] - e["mass_ic"][0])) <= 1e-13 * abs(m0)


def test_c4_tc5_config(P, oracle_mod):
    """C4 as BASELINE.json names it: Williamson TC5 (flow over the isolated
    mountain; an EXTENSION -- the reference has no orography, so this is
    parity against the oracle's restatement of the same source, 'parity
    unpinned' against the reference), p=4, 1440x720, 3 steps."""
    t, orc, X = oracle_mod.build_case("williamson_tc5", 1440, 720, 4)
    setup = P.build_case(P.default_config("williamson_tc5").override(nx=1440, ny=720, p=4))
    op = P.SpatialOperator(setup.mesh, 4, setup.model)
    st = op.project_state(setup.ic)
    assert np.array_equal(st.to_numpy(), X)
    rhs_gate(orc, X, op.assemble_rhs(st).to_numpy())
    U, status, _ = orc.rk_steps(X, 5e-4, 3, 3)
    assert status == 0
    m0 = P.mass_integral(st, op)
    op.ssprk3_steps(st, 5e-4, 3)
    assert op.status()[0] == 0
    gate_states(st.to_numpy(), U, X, "williamson_tc5")
    assert abs(P.mass_integral(st, op) - m0) <= 1e-13 * abs(m0)

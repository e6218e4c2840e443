"""GPU tests of the reference-facing API contract (round 2 additions):

* rk_step(state, op.assemble_rhs, dt, tableau(k)) runs as k stage kernels
  per step on the (lazily converted) nodal values and matches the Butcher
  form / the oracle;
* the modal single-launch entry points equal convert -> nodal -> convert;
* failure semantics: PositivityError leaves u^n in place (rk_step), and a
  fused integrate() batch restores the state the reference would leave,
  classifying the first failing step per status bit;
* ownership: no entry point allocates device memory after dgswe_create,
  misaligned state pointers are rejected;
* the bounded peer wait of the fused band exchange (PEER_TIMEOUT bit);
* the orography extension (TC5) against the oracle's restatement.
"""

import ctypes

import numpy as np
import pytest
import torch

from conftest import oracle_case

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2303_11767_b200 as P
    torch.cuda.set_device(0)
    return P


def rel(a, b, v):
    return float(np.linalg.norm(a[v] - b[v]) / max(np.linalg.norm(b[v]), 1e-300))


def make(P, case, nx, ny, p, nz=1, **kw):
    setup = P.build_case(P.default_config(case).override(nx=nx, ny=ny, p=p, nz=nz))
    return setup, P.SpatialOperator(setup.mesh, p, setup.model, nz=nz, **kw)


@pytest.mark.parametrize("order", [1, 2, 3, 4])
def test_rk_step_fused_vs_oracle(P, oracle_mod, order):
    """The reference's rk_step with tableau(k): k stage launches per step,
    equal to the oracle's Butcher steps (Shu-Osher vs Butcher: rounding);
    the state is read back (to_numpy) through the lazy nodal->modal
    conversion."""
    setup, op = make(P, "williamson_tc6", 40, 20, 3)
    t, orc, X = oracle_mod.build_case("williamson_tc6", 40, 20, 3)
    st = op.state_from_array(X)
    tab = P.tableau(order)
    ws = P.stepping._RKWorkspace(st, tab.s)
    dt = {1: 0.5, 2: 1.0, 3: 4.0, 4: 4.0}[order]
    n0 = op.launch_count()
    for _ in range(10):
        P.rk_step(st, op.assemble_rhs, dt, tab, ws)
    # one conversion (of a copy) to nodal values on the first call, then
    # only stage kernels (no copies, axpys or per-step conversions)
    assert op.launch_count() - n0 == 10 * order + 1
    U, status, _ = orc.rk_steps(X, dt, order, 10)
    assert status == 0
    got = st.to_numpy()
    for v in range(3):
        assert rel(got, U, v) <= 1e-12, (v, rel(got, U, v))
    b = op.state_from_array(X)                           # Butcher form: same steps
    for _ in range(10):
        P.rk_step(b, op.assemble_rhs, dt, tab, fused=False)
    for v in range(3):
        assert rel(got, b.to_numpy(), v) <= 1e-12


def test_modal_single_launch_equals_convert_path(P):
    """dgswe_stage / dgswe_stage2 / dgswe_rhs on modal states (one launch,
    in-kernel conversion) vs converting to nodal values, the nodal stage and
    converting back (rounding differs only in the output conversion)."""
    setup, op = make(P, "williamson_tc6", 70, 21, 3, nz=2)
    st = op.project_state(setup.ic)
    st.data[1] *= 1.0001
    w = op.zero_state()
    op.stage(0.0, None, 1.0, st, 7.0, w)
    y = op.zero_state()
    op.stage(0.75, st, 0.25, w, 1.75, y)                 # modal: one launch each
    c = op._ctx
    wn, un = w.copy(), st.copy()
    c.convert(wn.data, True, 0, 21)
    c.convert(un.data, True, 0, 21)
    yn = op.zero_state()
    c.set_basis(True)
    try:
        op.stage(0.75, un, 0.25, wn, 1.75, yn)
    finally:
        c.set_basis(False)
    c.convert(yn.data, False, 0, 21)
    d = (y.data - yn.data).abs().max().item()
    assert d <= 1e-13 * y.data.abs().max().item()
    k = op.assemble_rhs(st)
    k2 = op.zero_state()
    op.stage(0.0, None, 0.0, st, 1.0, k2)
    assert torch.equal(k.data, k2.data)
    acc = st.copy()
    y2 = op.zero_state()
    op.stage2(1.0, st, 0.0, w, 3.0, y2, acc, 0.5, acc)   # Y2 aliases A
    a = y2.data - st.data
    b2 = acc.data - st.data
    scale = k.data.abs().max().item()
    assert (a - 3.0 * op.assemble_rhs(w).data).abs().max().item() <= 1e-12 * scale * 3 + 1e-9
    assert (b2 - 0.5 * op.assemble_rhs(w).data).abs().max().item() <= 1e-12 * scale + 1e-9
    assert op.status()[0] == 0


def test_rk_step_positivity_leaves_state(P):
    """PositivityError from a stage RHS: state stays u^n (timestep.py:162,
    models.py:143-146), for the fused and the Butcher form."""
    setup, op = make(P, "williamson_tc6", 12, 6, 2)
    st = op.project_state(setup.ic)
    st.data[0, 3, 0, 0, 0, 5] = -100.0
    before = st.data.clone()
    for fused in (True, False):
        with pytest.raises(P.PositivityError):
            P.rk_step(st, op.assemble_rhs, 1.0, P.tableau(3), fused=fused)
        assert torch.equal(st.data, before)


def _crash_state(P):
    """TC6 at a stable dt with a patch of nearly dry cells whose momentum is
    kept: the 50x velocities drain them, h fails after a few steps."""
    setup, op = make(P, "williamson_tc6", 24, 12, 2)
    st = op.project_state(setup.ic)
    st.data[0, 5:7, 0, 0, :, 3:9] *= 0.02               # all h modes of a few cells
    return setup, op, st


@pytest.mark.parametrize("check", [None, "h"])
def test_integrate_failure_state_matches_unfused(P, check):
    """A failing step inside a fused batch: same step, time, message class
    and final state as the per-step (unfused) loop of the reference."""
    setup, op, st = _crash_state(P)
    ctl = P.TimeControls(2000.0, dt=10.0)
    ref = st.copy()
    with pytest.raises(P.DivergenceError) as e1:
        P.integrate(st, op, ctl, P.tableau(3), check_positivity=check, batch=16)
    with pytest.raises(P.DivergenceError) as e2:
        P.integrate(ref, op, ctl, P.tableau(3), check_positivity=check, fused=False)
    assert e1.value.step == e2.value.step and e1.value.t == e2.value.t
    assert ("cell-mean" in str(e1.value)) == ("cell-mean" in str(e2.value))
    a, b = st.to_numpy(), ref.to_numpy()
    if np.all(np.isfinite(b)):
        for v in range(3):
            assert rel(a, b, v) <= 1e-10, (v, rel(a, b, v))


def test_status_tags_per_bit(P):
    """The first failing step per status bit (one shared tag
    misclassified a cell-mean failure followed by a positivity failure)."""
    setup, op, st = _crash_state(P)
    op.status(reset=True)
    op.rk_steps(st, 10.0, 60, 3, check_mean=True)
    flags, tags = op.status_tags(reset=True)
    assert flags
    for b in range(4):
        if flags & (1 << b):
            assert 0 <= tags[b] < 60
        else:
            assert tags[b] == 2 ** 31 - 1


def test_no_device_allocation_after_create(P):
    """Every entry point runs on caller buffers and the context's
    create-time allocations: around a fresh context's first
    calls -- kernels already loaded by a first context -- free device
    memory is unchanged (round 1 allocated three state-sized scratch buffers
    inside the first modal stage call)."""
    def calls(setup, op, st, out, y, acc):
        op.assemble_rhs(st, out)
        op.stage(0.75, st, 0.25, out, 1.0, y)
        op.stage2(1.0, st, 0.0, out, 1.0, y, acc, 0.5, acc)
        op.axpy(1e-3, out, y)
        c = op._ctx
        P._lib.check(c.lib.dgswe_alpha_prepass(c.h, ctypes.c_void_p(st.data.data_ptr()), c.stream()), "alpha")
        P.mass_integral(st, op)
        op.status()

    bufs = []
    for _ in range(2):
        setup, op = make(P, "williamson_tc6", 512, 256, 3, rusanov=P.RusanovParams("global"))
        st = op.project_state(setup.ic)
        bufs.append((setup, op, st, op.zero_state(), op.zero_state(), op.zero_state()))
    calls(*bufs[0])                                       # loads every kernel module used
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    calls(*bufs[1])
    torch.cuda.synchronize()
    assert torch.cuda.mem_get_info()[0] == free0


def test_misaligned_state_rejected(P):
    setup, op = make(P, "williamson_tc6", 12, 6, 2)
    st = op.project_state(setup.ic)
    n = st.data.numel()
    raw = torch.zeros(n + 1, dtype=torch.float64, device="cuda")
    view = raw[1:]                                        # 8-byte offset
    c = op._ctx
    rc = c.lib.dgswe_rhs(c.h, ctypes.c_void_p(view.data_ptr()), ctypes.c_void_p(st.data.data_ptr()),
                         c.stream())
    assert rc == -1 and b"aligned" in c.lib.dgswe_last_error()
    with pytest.raises(ValueError):
        P.State(view.view(st.data.shape), 12, 6, 1, op.nphi)


def test_peer_wait_times_out(P):
    """A band launch whose neighbour never delivers: bounded wait, the
    PEER_TIMEOUT status bit, no hung GPU (the band is row0 > 0, so it waits
    for its southern halo; the receive counter never moves)."""
    from paper_2303_11767_b200.bands import BandLayout, BandOperator
    setup, op = make(P, "williamson_tc6", 48, 16, 3)
    L = BandLayout(16, 2, 1)
    bop = BandOperator(op, L, transport="p2p")
    c = bop.ctx
    ctrl = torch.zeros(4, dtype=torch.int64, device="cuda")
    ctrl[2] = 1                                            # one edge stage "completed": needs deliveries
    base = ctrl.data_ptr()
    P._lib.check(c.lib.dgswe_set_exchange(c.h, 0, None, 0, None, ctypes.c_void_p(base),
                                          ctypes.c_void_p(base + 16)), "set_exchange")
    P._lib.check(c.lib.dgswe_set_peer_timeout(c.h, 20_000_000), "set_peer_timeout")   # 20 ms
    u, y = bop.empty(), bop.empty()
    u[:, :, 0] = 1000.0                                    # positive h
    c.set_basis(True)
    try:
        P._lib.check(c.lib.dgswe_stage_band(c.h, 0.0, None, 1.0, ctypes.c_void_p(u.data_ptr()), 1.0,
                                            ctypes.c_void_p(y.data_ptr()), 0, None, None, c.stream()),
                     "stage_band")
        flags, tags = c.status_tags()
    finally:
        c.set_basis(False)
    assert flags & P._lib.STATUS_PEER_TIMEOUT
    assert tags[3] == 0


@pytest.mark.parametrize("p", [2, 4])
def test_tc5_orography_vs_oracle(P, oracle_mod, p):
    """Williamson TC5 (EXTENSION, parity unpinned against the reference):
    one RHS and 5 steps vs the oracle's restatement of the orography source,
    modal (assemble_rhs, rk_step) and nodal (rk_steps) kernel variants."""
    nx, ny = 36, 18
    t, orc, X = oracle_mod.build_case("williamson_tc5", nx, ny, p)
    setup, op = make(P, "williamson_tc5", nx, ny, p)
    st = op.project_state(setup.ic)
    assert np.array_equal(st.to_numpy(), X)
    K = op.assemble_rhs(st).to_numpy()
    Kr = orc.rhs(X)
    rng = np.random.default_rng(0)
    Kp = orc.rhs(X * (1.0 + rng.integers(-1, 2, size=X.shape) * 2.0 ** -52))
    for v in range(3):
        sens = float(np.linalg.norm(Kp[v] - Kr[v]) / np.linalg.norm(Kr[v]))
        assert rel(K, Kr, v) <= max(20 * sens, 1e-13), (v, rel(K, Kr, v), sens)
    # the mountain matters: the same state without orography gives another RHS
    t0, orc0, _ = oracle_mod.build_case("williamson_tc2", nx, ny, p)
    assert rel(orc0.rhs(X), Kr, 1) > 1e-6
    dt = 8.0 if p == 2 else 2.0
    U, status, _ = orc.rk_steps(X, dt, 3, 5)
    assert status == 0
    a = op.state_from_array(X)
    op.rk_steps(a, dt, 5, 3)
    b = op.state_from_array(X)
    for _ in range(5):
        P.rk_step(b, op.assemble_rhs, dt, P.tableau(3))
    assert op.status()[0] == 0
    mom = np.sqrt(np.linalg.norm(U[1]) ** 2 + np.linalg.norm(U[2]) ** 2)
    for got in (a.to_numpy(), b.to_numpy()):
        assert rel(got, U, 0) <= 1e-11 and rel(got, U, 1) <= 1e-11
        assert np.linalg.norm(got[2] - U[2]) / mom <= 1e-11

"""Explicit SSP Runge-Kutta stepping and the integration loop.

Same API as /root/reference/pkg/src/dgswe/timestep.py (``ButcherTableau``,
``tableau``, ``TimeControls``, ``DivergenceError``, ``StepLog``,
``rk_step``, ``integrate``).  Two device paths:

* ``rk_step`` -- with ``tableau(1..4)`` one stage kernel per stage
  (Shu-Osher / RK4-accumulator forms) on the state's nodal values: the
  state is converted in place on the first call and stays nodal until it
  is read (``State.data`` converts back); any other
  tableau (or ``fused=False``) in Butcher form: per stage a device copy,
  axpy launches (two roundings, like ``_axpy`` timestep.py:132-141) and one
  RHS launch.  One status read per step.
* ``integrate`` with ``tableau(1..4)`` -- the tableaux of timestep.py:57-82
  evaluated as fused stages (RHS + stage combination in one kernel):
  Euler; Heun and SSPRK3 in Shu-Osher form (SSPRK3: three launches per step,
  21.3 B/DOF of HBM traffic); classical RK4 with its accumulator as the
  stage kernel's second output.  Steps are batched into CUDA graphs; status
  (positivity / non-finite / cell-mean) is read once per batch and mapped
  back to the failing step.  Stage and Butcher forms are the same methods;
  they differ only in rounding (~1e-15 relative after 100 steps, SURVEY.md
  section 8a10).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

from . import _lib
from .geometry import min_effective_diameter
from .physics import PositivityError


class DivergenceError(RuntimeError):
    """Integration produced a non-finite or invalid state."""

    def __init__(self, message, step, t):
        super().__init__(f"{message} (step {step}, t={t:.6g})")
        self.step = step
        self.t = t


@dataclass(frozen=True)
class ButcherTableau:
    s: int
    a: tuple
    b: tuple
    c: tuple

    def __post_init__(self):
        if not (len(self.a) == len(self.b) == len(self.c) == self.s):
            raise ValueError("tableau dimensions inconsistent with stage count")
        for i, row in enumerate(self.a):
            if len(row) != self.s:
                raise ValueError("tableau matrix must be square")
            if any(x != 0.0 for x in row[i:]):
                raise ValueError("tableau must be strictly lower triangular")
            if abs(sum(row) - self.c[i]) > 1e-14:
                raise ValueError("abscissae must equal the stage row sums")
        if abs(sum(self.b) - 1.0) > 1e-14:
            raise ValueError("stage weights must sum to one")


# the paper's Table 1 (timestep.py:57-82)
_TABLES = {
    1: ButcherTableau(1, ((0.0,),), (1.0,), (0.0,)),
    2: ButcherTableau(2, ((0.0, 0.0), (1.0, 0.0)), (0.5, 0.5), (0.0, 1.0)),
    3: ButcherTableau(3, ((0.0, 0.0, 0.0), (1.0, 0.0, 0.0), (0.25, 0.25, 0.0)),
                      (1.0 / 6.0, 1.0 / 6.0, 2.0 / 3.0), (0.0, 1.0, 0.5)),
    4: ButcherTableau(4, ((0.0, 0.0, 0.0, 0.0), (0.5, 0.0, 0.0, 0.0), (0.0, 0.5, 0.0, 0.0),
                          (0.0, 0.0, 1.0, 0.0)),
                      (1.0 / 6.0, 1.0 / 3.0, 1.0 / 3.0, 1.0 / 6.0), (0.0, 0.5, 0.5, 1.0)),
}


def tableau(order: int) -> ButcherTableau:
    try:
        return _TABLES[int(order)]
    except KeyError:
        raise ValueError(f"unsupported RK order {order}; choose 1..4") from None


@dataclass(frozen=True)
class TimeControls:
    """dt directly, or dt = courant * H / (max(p,1) * c_max) from the
    initial state (timestep.py:93-121).  The reference's Courant rule is
    not a stable bound on this mesh; prefer dt."""

    t_final: float
    dt: float | None = None
    courant: float | None = None

    def __post_init__(self):
        if (self.dt is None) == (self.courant is None):
            raise ValueError("specify exactly one of dt or courant")
        if self.dt is not None and self.dt <= 0:
            raise ValueError("dt must be positive")
        if self.courant is not None and self.courant <= 0:
            raise ValueError("courant number must be positive")
        if self.t_final < 0:
            raise ValueError("t_final must be non-negative")

    def resolve_dt(self, diameter: float, p: int, c_max: float) -> float:
        if self.dt is not None:
            return self.dt
        if c_max <= 0:
            raise ValueError("cannot derive dt from a zero wavespeed")
        return self.courant * diameter / (max(p, 1) * c_max)


@dataclass
class StepLog:
    steps: int = 0
    t: float = 0.0
    dt: float = 0.0
    wall_seconds: float = 0.0
    c_max: float = 0.0
    diameter: float = 0.0


class _RKWorkspace:
    def __init__(self, state, stages: int):
        self.stage_input = state.copy()
        self.k = [state.copy() for _ in range(stages)]
        self.spare = state.copy()   # fused rk_step: nodal copy of a modal u^n (first step)


def _device_operator(rhs_fn):
    """The SpatialOperator behind ``rhs_fn`` if it is one's assemble_rhs."""
    from .operator import SpatialOperator
    op = getattr(rhs_fn, "__self__", None)
    if isinstance(op, SpatialOperator) and getattr(rhs_fn, "__func__", None) is \
            SpatialOperator.assemble_rhs:
        return op
    return None


def _fused_order(tab: ButcherTableau):
    """The order k if ``tab`` is tableau(k) (fused stage form exists), else None."""
    for k, t in _TABLES.items():
        if tab == t:
            return k
    return None


def rk_step(state, rhs_fn, dt: float, tab: ButcherTableau, workspace: _RKWorkspace | None = None,
            fused: bool = True):
    """One explicit RK step, updating ``state`` in place (timestep.py:149-167).

    With our operator's ``assemble_rhs`` and ``tableau(1..4)`` (``fused``):
    one stage kernel per stage on the state's nodal values (the stage
    combination fused into the RHS kernel: SSPRK3 moves 21.3 B/DOF instead
    of the Butcher form's copies and axpys; the state is converted to nodal
    values once and back only when something reads it), the new state
    written into a workspace buffer that is swapped into ``state`` on
    success.  Otherwise
    (or ``fused=False``) the Butcher form of the reference: per stage a
    copy, axpys with two roundings and one RHS launch.  Both read the status
    once per step: PositivityError (from any stage's RHS) leaves ``state``
    at u^n like the reference; DivergenceError (non-finite update) is raised
    after the update, as the reference's finite check does.
    """
    ws = workspace or _RKWorkspace(state, tab.s)
    op = _device_operator(rhs_fn)
    if op is None:
        return _rk_step_generic(state, rhs_fn, dt, tab, ws)
    order = _fused_order(tab) if fused else None
    if order is not None:
        bufs = [ws.stage_input] + list(ws.k) + [ws.spare]
        new = op.rk_step_fused(state, dt, order, bufs)
        flags, _ = op.status(reset=True)
        op.raise_on_status(flags)                   # PositivityError: state still u^n
        # the new (nodal) state becomes ``state``; its old buffer joins the workspace
        slot = next(b for b in bufs if b._data is new)
        state._data, slot._data = new, state._data
        state._nodal, slot._nodal = op, None
        if flags & _lib.STATUS_NONFINITE:
            raise DivergenceError("non-finite state after RK update", -1, float("nan"))
        return state
    for i in range(tab.s):
        ws.stage_input.data.copy_(state.data)      # u * 1.0 is exact
        for j in range(i):
            coef = dt * tab.a[i][j]
            if coef != 0.0:
                op.axpy(coef, ws.k[j], ws.stage_input)
        op.assemble_rhs(ws.stage_input, out=ws.k[i], check=False)
    flags, _ = op.status(reset=True)               # before the update: u^n stays on error
    op.raise_on_status(flags)
    last = max((i for i in range(tab.s) if dt * tab.b[i] != 0.0), default=-1)
    for i in range(tab.s):
        coef = dt * tab.b[i]
        if coef != 0.0:
            op.axpy(coef, ws.k[i], state, check_finite=(i == last))
    flags, _ = op.status(reset=True)
    if flags & _lib.STATUS_NONFINITE or last < 0 and not math.isfinite(state.max_abs()):
        raise DivergenceError("non-finite state after RK update", -1, float("nan"))
    return state


def _rk_step_generic(state, rhs_fn, dt, tab, ws):
    """Any callable rhs_fn(state, out=...) on device states (torch ops)."""
    for i in range(tab.s):
        ws.stage_input.data.copy_(state.data)
        for j in range(i):
            coef = dt * tab.a[i][j]
            if coef != 0.0:
                ws.stage_input.data.add_(ws.k[j].data * coef)
        rhs_fn(ws.stage_input, out=ws.k[i])
    for i in range(tab.s):
        coef = dt * tab.b[i]
        if coef != 0.0:
            state.data.add_(ws.k[i].data * coef)
    if not math.isfinite(state.max_abs()):
        raise DivergenceError("non-finite state after RK update", -1, float("nan"))
    return state


def _step_sizes(t_final: float, dt: float):
    """Per-step dt and end time exactly as the reference loop forms them
    (timestep.py:205-219)."""
    n = max(1, math.ceil(t_final / dt - 1e-12))
    t = 0.0
    out = []
    for step in range(1, n + 1):
        h = min(dt, t_final - t)
        t_next = t_final if step == n else t + h
        out.append((h, t, t_next))
        t = t_next
    return out


def integrate(state, operator, controls: TimeControls, tab: ButcherTableau, callbacks=(),
              check_positivity=None, batch: int = 64, fused: bool = True):
    """Advance ``state`` to t_final (timestep.py:180-233).

    With our SpatialOperator and ``tableau(1..4)`` the steps run as fused
    CUDA-graph batches of up to ``batch`` steps between callback
    cadences; errors are detected per batch and reported with the exact
    failing step and time, as the reference does per step, and ``state``
    is left where the reference leaves it: a batch starts from a snapshot,
    and on failure the state is restored and re-advanced to the step before
    the failing one (non-positive / non-finite) or through it (cell mean,
    which the reference checks after the update).  ``fused=False`` steps
    with the Butcher-form ``rk_step`` (the reference's operation order).
    """
    log = StepLog()
    log.diameter = min_effective_diameter(operator.mesh)
    c_max = operator.max_physical_speed(state)
    log.c_max = c_max
    dt = controls.resolve_dt(log.diameter, operator.p, c_max)
    log.dt = dt
    t_final = controls.t_final
    for _, fn in callbacks:
        fn(0, 0.0, state)
    if t_final == 0.0:
        return state, log

    steps = _step_sizes(t_final, dt)
    n_steps = len(steps)
    from .operator import SpatialOperator
    order = _fused_order(tab)
    use_fused = (fused and isinstance(operator, SpatialOperator) and order is not None
                 and check_positivity in (None, "h"))
    started = time.perf_counter()
    if not use_fused:
        ws = _RKWorkspace(state, tab.s)
        for step, (h, t0, t1) in enumerate(steps, start=1):
            try:
                rk_step(state, operator.assemble_rhs, h, tab, ws, fused=False)
            except (PositivityError, DivergenceError) as exc:
                log.steps, log.t = step - 1, t0
                log.wall_seconds = time.perf_counter() - started
                raise DivergenceError(str(exc), step, t0) from exc
            if check_positivity is not None:
                means = state.interior_coeffs(check_positivity)[..., 0]
                if not float(means.min()) > 0.0:
                    log.steps, log.t = step, t1
                    raise DivergenceError(f"cell-mean {check_positivity} lost positivity", step, t1)
            for cadence, fn in callbacks:
                if step % cadence == 0 or step == n_steps:
                    fn(step, t1, state)
        log.steps, log.t = n_steps, steps[-1][2]
        log.wall_seconds = time.perf_counter() - started
        return state, log

    cadences = [c for c, _ in callbacks]
    step = 0
    operator.status(reset=True)
    snapshot = state.data.clone()
    check_mean = check_positivity == "h"
    while step < n_steps:
        h = steps[step][0]
        k = 1
        while step + k < n_steps and k < batch and steps[step + k][0] == h:
            if any((step + k) % c == 0 for c in cadences):
                break
            k += 1
        snapshot.copy_(state.data)
        operator.rk_steps(state, h, k, order, check_mean=check_mean)
        flags, tags = operator.status_tags(reset=True)
        if flags:
            # the earliest failing step decides; at equal steps the RHS
            # positivity check precedes the finite check, which precedes the
            # cell-mean check (timestep.py:162-166, 220-226)
            tag, bit = min((tags[b], b) for b in range(_lib.STATUS_BITS) if flags & (1 << b))
            bad = step + tag + 1
            t0, t1 = steps[bad - 1][1], steps[bad - 1][2]
            mean = (1 << bit) == _lib.STATUS_MEAN_NONPOS
            state.data.copy_(snapshot)
            redo = bad - step if mean else bad - 1 - step
            if redo > 0:
                operator.rk_steps(state, h, redo, order)
                operator.status(reset=True)
            log.wall_seconds = time.perf_counter() - started
            if mean:
                log.steps, log.t = bad, t1
                raise DivergenceError("cell-mean h lost positivity", bad, t1)
            log.steps, log.t = bad - 1, t0
            what = ("non-positive water height at a quadrature node"
                    if (1 << bit) == _lib.STATUS_POSITIVITY else "non-finite state after RK update")
            raise DivergenceError(what, bad, t0)
        step += k
        for cadence, fn in callbacks:
            if step % cadence == 0 or step == n_steps:
                fn(step, steps[step - 1][2], state)
    log.steps, log.t = n_steps, steps[-1][2]
    log.wall_seconds = time.perf_counter() - started
    return state, log

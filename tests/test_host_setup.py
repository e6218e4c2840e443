"""Host-side setup of the product package (geometry, tableaux, controls,
cases): bit-identical to the reference fixtures, same validation errors."""

import math

import numpy as np
import pytest

import paper_2303_11767_b200 as P
from paper_2303_11767_b200 import geometry as G
from paper_2303_11767_b200.stepping import _step_sizes


def _tag_shape(tag):
    nx, rest = tag[len("tab_"):].split("x")
    ny, p = rest.split("_p")
    return int(nx), int(ny), int(p)


def test_vander_and_mass_tables_bit_identical(golden):
    meta, g = golden
    for tag in meta["tables"]:
        nx, ny, p = _tag_shape(tag)
        mesh = P.build_latlon_mesh(nx, ny)
        quad = P.gauss_legendre(p + 1)
        v = P.build_vander(p, quad)
        assert np.array_equal(quad.nodes, g[f"{tag}/nodes"])
        assert np.array_equal(quad.weights, g[f"{tag}/weights"])
        assert np.array_equal(v.phi, g[f"{tag}/phi"])
        assert np.array_equal(v.grad_x, g[f"{tag}/grad_x"])
        assert np.array_equal(v.grad_y, g[f"{tag}/grad_y"])
        for e in range(4):
            assert np.array_equal(v.edges[e], g[f"{tag}/edge{e}"]), (tag, e)
        M, Minv = P.sphere_row_mass_matrices(p, mesh, quad)
        assert np.array_equal(M, g[f"{tag}/M_rows"])
        assert np.array_equal(Minv, g[f"{tag}/Minv"])
        # the device coordinate tables (operator._Context) use these formulas
        th = G.node_latitudes(mesh, quad.nodes)
        R = G.EARTH.radius
        ref = g[f"{tag}/coords_xe.cos_over_r"][1:ny + 1].reshape(th.shape)
        assert np.array_equal(np.cos(th) / R, ref)
        ref = g[f"{tag}/coords_int.sin_over_r"][1:ny + 1].reshape(ny, p + 1, p + 1)[:, 0, :]
        assert np.array_equal(np.sin(th) / R, ref)
        fc = 2.0 * G.EARTH.omega * np.sin(th) * np.cos(th)
        ref = g[f"{tag}/coords_int.f_cos"][1:ny + 1].reshape(ny, p + 1, p + 1)[:, 0, :]
        assert np.array_equal(fc, ref)
        yb = g[f"{tag}/coords_yb.cos_over_r"][1:ny + 1]
        yt = g[f"{tag}/coords_yt.cos_over_r"][1:ny + 1]
        edge = np.cos(mesh.y_edges) / R
        assert np.array_equal(edge[:-1], yb) and np.array_equal(edge[1:], yt)


@pytest.mark.parametrize("name", ["tc2_c1", "tc6_p0", "tc6_p3", "tc6_p5", "tc2_p3_odd", "tc6_ny1",
                                  "tc2_nx1", "tc6_wide"])
def test_projection_bit_identical(golden, name):
    meta, g = golden
    e = meta["cases"][name]
    cfg = P.default_config(e["case"]).override(nx=e["nx"], ny=e["ny"], p=e["p"])
    setup = P.build_case(cfg)
    quad = P.gauss_legendre(e["p"] + 1)
    v = P.build_vander(e["p"], quad)
    stack = np.stack([P.project_initial(setup.ic[n], setup.mesh, v) for n in ("h", "hu", "hv")])
    assert np.array_equal(stack, g[f"{name}/ic"][:, :, :, 0, :])


def test_mesh_api():
    m = P.build_latlon_mesh(8, 4)
    assert m.dx == float(m.x_edges[1] - m.x_edges[0])
    assert m.neighbor(0, 1, P.LEFT) == G.NeighborRef("periodic_wrap", (7, 1))
    assert m.neighbor(7, 1, P.RIGHT) == G.NeighborRef("periodic_wrap", (0, 1))
    assert m.neighbor(3, 0, P.BOTTOM).kind == "pole_closed"
    assert m.neighbor(3, 3, P.TOP).kind == "pole_closed"
    assert m.neighbor(3, 2, P.TOP) == G.NeighborRef("interior", (3, 3))
    with pytest.raises(ValueError):
        P.build_latlon_mesh(0, 4)
    with pytest.raises(ValueError):
        m.neighbor(0, 0, 7)
    # pole rows use the equator-side edge (mesh.py:155-174)
    R = m.radius
    expect = min(min(R * m.dy, R * max(math.cos(m.y_edges[j]), math.cos(m.y_edges[j + 1])) * m.dx
                     if min(math.cos(m.y_edges[j]), math.cos(m.y_edges[j + 1])) <= 1e-14 else
                     min(R * m.dy, R * min(math.cos(m.y_edges[j]), math.cos(m.y_edges[j + 1])) * m.dx))
                 for j in range(m.ny))
    assert P.min_effective_diameter(m) == expect


def test_tableaux_and_controls():
    t3 = P.tableau(3)
    assert t3.b == (1.0 / 6.0, 1.0 / 6.0, 2.0 / 3.0) and t3.a[2] == (0.25, 0.25, 0.0)
    assert P.tableau(4).c == (0.0, 0.5, 0.5, 1.0)
    with pytest.raises(ValueError):
        P.tableau(5)
    with pytest.raises(ValueError):
        P.ButcherTableau(2, ((0.0, 1.0), (1.0, 0.0)), (0.5, 0.5), (1.0, 1.0))
    with pytest.raises(ValueError):
        P.ButcherTableau(1, ((0.0,),), (0.9,), (0.0,))
    with pytest.raises(ValueError):
        P.TimeControls(1.0)
    with pytest.raises(ValueError):
        P.TimeControls(1.0, dt=1.0, courant=0.1)
    with pytest.raises(ValueError):
        P.TimeControls(1.0, dt=-1.0)
    with pytest.raises(ValueError):
        P.TimeControls(-1.0, dt=1.0)
    assert P.TimeControls(1.0, courant=0.5).resolve_dt(10.0, 3, 2.0) == 0.5 * 10.0 / (3 * 2.0)
    with pytest.raises(ValueError):
        P.TimeControls(1.0, courant=0.5).resolve_dt(10.0, 3, 0.0)


def test_step_schedule_matches_reference_loop():
    """integrate's per-step dt and t (timestep.py:205-219)."""
    for t_final, dt in ((10.0, 3.0), (1.0, 0.1), (100.0, 7.0), (0.3, 1.0)):
        n = max(1, math.ceil(t_final / dt - 1e-12))
        t, ref = 0.0, []
        for step in range(1, n + 1):
            h = min(dt, t_final - t)
            t_next = t_final if step == n else t + h
            ref.append((h, t, t_next))
            t = t_next
        assert _step_sizes(t_final, dt) == ref


def test_cases_api():
    cfg = P.default_config("williamson_tc6")
    assert (cfg.nx, cfg.ny, cfg.p, cfg.rk, cfg.dt) == (40, 20, 3, 4, 4.0)
    assert cfg.override(nx=8, dt=None).nx == 8
    with pytest.raises(ValueError):
        P.default_config("nope")
    setup = P.build_case(P.default_config("advection_sine"))
    assert setup.model.beta == (1.0, 1.0) and setup.mesh.kind == "planar" and setup.mesh.dx == 0.05
    setup = P.build_case(P.default_config("williamson_tc2"))
    assert setup.model.h_floor == 1e-8 * (2.94e4 / 9.81)
    assert setup.exact(123.0) is not None


def test_rusanov_params():
    with pytest.raises(ValueError):
        P.RusanovParams("bogus")
    assert P.RusanovParams().mode == "local"


def test_op_recorder_hook():
    """set_op_recorder (fields.py:66-76) mirror: entries carry the launch
    region, analytic flops and algorithmic bytes; None clears the hook."""
    import paper_2303_11767_b200 as P
    from paper_2303_11767_b200 import tracing

    class Rec:
        def __init__(self):
            self.rows = []

        def record(self, kind, op, rgn, flops, nbytes):
            self.rows.append((kind, op, rgn, flops, nbytes))

    rec = Rec()
    P.set_op_recorder(rec)
    try:
        rgn = tracing.LaunchRegion((720, 360, 1), 3)
        tracing.record("stage", "dgswe_stage", rgn, 24.0, tracing.stage_flops_per_dof(3))
    finally:
        P.set_op_recorder(None)
    tracing.record("stage", "ignored", rgn, 16.0, 1.0)      # no recorder: nothing happens
    assert len(rec.rows) == 1
    kind, op, r, flops, nbytes = rec.rows[0]
    assert (kind, op) == ("stage", "dgswe_stage") and r.dofs == 720 * 360 * 48
    assert nbytes == 24 * r.dofs and flops > 20 * r.dofs

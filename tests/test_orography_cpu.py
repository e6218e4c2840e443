"""Orography extension (Williamson TC5; the reference has none):
the oracle's source factors and the host-side model/case plumbing, on CPU.

The factors are -(g/R) db/dlambda and -(g cos/R) db/dtheta at the interior
Gauss nodes, grad b taken from b's degree-p nodal interpolant -- exact for a
bottom that is a polynomial of degree <= p in each element coordinate."""

import numpy as np
import pytest


@pytest.mark.parametrize("p", [1, 2, 4])
def test_factors_exact_for_polynomial_bottom(oracle_mod, p):
    O = oracle_mod
    t = O.make_tables(10, 6, p, O.TC5_H0)
    ox, oy = O.orography_factors(t, lambda lam, th: lam * th + 3.0 * th)
    x, y = O.node_coords(t, t.nodes)
    n = p + 1
    lam = np.broadcast_to(x[:, None, :, None], (t.nx, t.ny, n, n)).reshape(t.nx, t.ny, n * n)
    th = np.broadcast_to(y[None, :, None, :], (t.nx, t.ny, n, n)).reshape(t.nx, t.ny, n * n)
    g_r = O.GRAVITY / O.RADIUS
    assert np.allclose(ox, -g_r * th, rtol=1e-12, atol=1e-18)
    assert np.allclose(oy, -g_r * np.cos(th) * (lam + 3.0), rtol=1e-12, atol=1e-18)


def test_flat_bottom_is_the_reference_model(oracle_mod):
    O = oracle_mod
    t, orc, X = O.build_case("williamson_tc2", 12, 6, 3)
    flat = O.Oracle(t, lambda lam, th: 0.0 * lam + 0.0 * th)
    assert np.array_equal(flat.rhs(X), orc.rhs(X))


def test_tc5_case_plumbing(oracle_mod):
    import paper_2303_11767_b200 as P
    O = oracle_mod
    cfg = P.default_config("williamson_tc5")
    assert cfg.case in P.CASE_IDS and cfg.p == 4
    setup = P.build_case(cfg.override(nx=36, ny=18, p=2))
    assert setup.model.bottom is P.tc5_bottom
    assert setup.model.h_floor == 1e-8 * O.TC5_H0
    lam = np.linspace(0.0, 2 * np.pi, 50)[:, None]
    th = np.linspace(-1.5, 1.5, 40)[None, :]
    for k in ("h", "hu", "hv"):
        assert np.array_equal(np.broadcast_to(setup.ic[k](lam, th), (50, 40)),
                              np.broadcast_to(O.ic_tc5()[k](lam, th), (50, 40)))
    b = P.tc5_bottom(lam, th)
    assert b.min() == 0.0 and b.max() > 0.0
    assert P.tc5_bottom(1.5 * np.pi, np.pi / 6) == 2000.0      # the cone's apex (Williamson 3.5)
    # the host projection is the oracle's (bitwise), as for the reference's cases
    t, orc, X = O.build_case("williamson_tc5", 36, 18, 2)
    got = np.stack([P.project_initial(setup.ic[k], setup.mesh, P.build_vander(2, P.gauss_legendre(3)))
                    for k in ("h", "hu", "hv")])
    assert np.array_equal(got[:, :, :, None, :], X)

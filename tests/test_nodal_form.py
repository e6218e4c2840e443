"""CPU check of the algebra behind the stage kernel's nodal form (DESIGN.md
section 3, "Nodal form of the reference's operator").

The kernel carries the state at the (p+1)^2 Gauss nodes and applies

    u'_ij = 1/(determ cos_j) [ c_x sum_k dh_ik F_kj + c_y sum_k dh_jk G_ik + c_s S_ij
                               + bd_y (mu_i fL_j - mu_(n-1-i) fR_j)
                               + bd_x (mu_j fB_i - mu_(n-1-j) fT_i) ]

with the tables of dgswe_b200.cu (dgswe_create): lm_i = l_i(-1),
mu_i = lm_i / w_i, dh_ik = w_k l_i'(x_k) / w_i, built from the Legendre
tables as l_i(x) = sum_a (2a+1)/2 w_i P_a(x_i) P_a(x).  Here that formula is
checked against the reference's modal operator, term by term, with the
package's own basis matrices (geometry.py, pinned to the reference's
golden tables in test_host_setup.py):

    u' = V M^-1 [ (determ/bd_x) grad_x^T (w F) + (determ/bd_y) grad_y^T (w G)
                  + determ phi^T (w S) - bnd ]          (dg.py:196-213, 455-502)

with V = phi (modal -> nodal) and the cos-weighted row mass matrix
(basis.py:159-177).  Exact in real arithmetic; the test allows rounding.
"""

import numpy as np
import pytest

from paper_2303_11767_b200.geometry import build_vander, gauss_legendre, legendre_deriv, legendre_eval


def nodal_tables(p):
    """The kernel's NodTab, restated (dgswe_b200.cu, dgswe_create)."""
    n = p + 1
    q = gauss_legendre(n)
    x, w = q.nodes, q.weights
    P = np.array([[legendre_eval(a, xi) for xi in x] for a in range(n)])      # P[a][q]
    D = np.array([[legendre_deriv(a, xi) for xi in x] for a in range(n)])     # P'[a][q]
    cf = 0.5 * (2 * np.arange(n) + 1)
    lm = np.array([sum(cf[a] * w[i] * P[a, i] * (-1) ** a for a in range(n)) for i in range(n)])
    dh = np.array([[sum(cf[a] * P[a, i] * w[k] * D[a, k] for a in range(n)) for k in range(n)]
                   for i in range(n)])
    return x, w, lm, lm / w, dh


@pytest.mark.parametrize("p", [0, 1, 2, 3, 4, 5])
def test_nodal_operator_equals_modal(p):
    rng = np.random.default_rng(p)
    n = p + 1
    quad = gauss_legendre(n)
    v = build_vander(p, quad)
    x, w1, lm, mu, dh = nodal_tables(p)
    # one latitude row of a lat-lon element: theta in [tb, tt], lambda width dlam
    tb, tt, dlam = 0.31, 0.36, 0.05
    determ = dlam * (tt - tb) / 4.0
    bdx, bdy = dlam / 2.0, (tt - tb) / 2.0
    cos_q = np.cos(0.5 * (tb + tt) + 0.5 * (tt - tb) * x)                   # per eta node j
    w2 = v.w                                                                # w_i w_j, q = i n + j
    M = determ * (v.phi.T * np.outer(w1, w1 * cos_q).reshape(-1)) @ v.phi
    Minv = np.linalg.inv(M)

    F, G, S = (rng.standard_normal((n, n)) for _ in range(3))               # nodal [i][j]
    fL, fR, fB, fT = (rng.standard_normal(n) for _ in range(4))             # face fluxes f*
    modal = ((determ / bdx) * v.grad_x.T @ (w2 * F.reshape(-1))
             + (determ / bdy) * v.grad_y.T @ (w2 * G.reshape(-1))
             + determ * v.phi.T @ (w2 * S.reshape(-1)))
    # boundary terms: outward-normal signs of dg.py:206-212 (LEFT/BOTTOM negative)
    e = v.edges
    bnd = (bdy * e[1].T @ (v.w_edge * fR) - bdy * e[0].T @ (v.w_edge * fL)
           + bdx * e[3].T @ (v.w_edge * fT) - bdx * e[2].T @ (v.w_edge * fB))
    want = (v.phi @ (Minv @ (modal - bnd))).reshape(n, n)

    rj = 1.0 / (determ * cos_q)
    acc = ((determ / bdx) * dh @ F                                           # sum_k dh_ik F_kj
           + (determ / bdy) * G @ dh.T                                       # sum_k dh_jk G_ik
           + determ * S
           + bdy * (np.outer(mu, fL) - np.outer(mu[::-1], fR))
           + bdx * (np.outer(fB, mu) - np.outer(fT, mu[::-1])))
    got = acc * rj[None, :]
    scale = np.abs(want).max()
    assert np.abs(got - want).max() <= 1e-11 * scale, np.abs(got - want).max() / scale


@pytest.mark.parametrize("p", [0, 1, 3, 6])
def test_nodal_traces_and_conversion(p):
    """Traces of the nodal tile (lm, reflected for +1) equal the modal edge
    evaluation (basis.py edges), and the two conversion formulas of
    convert_kernel are inverse to each other."""
    rng = np.random.default_rng(10 + p)
    n = p + 1
    quad = gauss_legendre(n)
    v = build_vander(p, quad)
    x, w, lm, mu, dh = nodal_tables(p)
    c = rng.standard_normal(n * n)
    u = (v.phi @ c).reshape(n, n)                                            # u[i][j]
    assert np.allclose(lm @ u, v.edges[0] @ c, rtol=0, atol=1e-12)         # left  (xi = -1)
    assert np.allclose(lm[::-1] @ u, v.edges[1] @ c, rtol=0, atol=1e-12)   # right (xi = +1)
    assert np.allclose(u @ lm, v.edges[2] @ c, rtol=0, atol=1e-12)         # bottom
    assert np.allclose(u @ lm[::-1], v.edges[3] @ c, rtol=0, atol=1e-12)   # top
    P = np.array([[legendre_eval(a, xi) for xi in x] for a in range(n)])
    wp = P * w[None, :]
    norm = np.outer(2 * np.arange(n) + 1, 2 * np.arange(n) + 1) / 4.0
    back = norm * (wp @ u @ wp.T)                                            # convert_kernel<P, false>
    assert np.allclose(back.reshape(-1), c, rtol=0, atol=1e-12)

"""Conservation and accuracy monitors used as parity gates.

``mass_integral`` and ``l2_error`` keep the reference's signatures and
reduction order (/root/reference/pkg/src/dgswe/diagnostics.py:42-107):
per-element contributions, then a sequential sum in ascending element
order, so printed digits are reproducible.  They run on a host copy of the
state (device versions are SURVEY.md section 8f rank 1).
"""

from __future__ import annotations

import math

import numpy as np

from .geometry import build_vander, element_node_coords, gauss_legendre


def _ordered_sum(cell: np.ndarray) -> float:
    total = 0.0
    for v in cell.reshape(-1):    # (nx, ny) C order == i-major, j-minor
        total += v
    return total


def mass_integral(state, op, var: str | None = None, level: int = 0) -> float:
    """Sum over elements of (M_j c)_0, the cos-weighted integral of var."""
    var = var or state.names[0]
    coeffs = state.interior_coeffs(var)[:, :, level, :]
    cell = np.einsum("ym,xym->xy", op.M_rows[:, 0, :], coeffs)
    return _ordered_sum(cell)


def l2_error(state, reference_fn, op, var: str | None = None, relative: bool = False,
             level: int = 0) -> float:
    """L2 norm of (numerical - reference) with a p+2 Gauss rule and the
    cos(theta) metric."""
    mesh = op.mesh
    var = var or state.names[0]
    quad = gauss_legendre(op.p + 2)
    vander = build_vander(op.p, quad)
    n = quad.n_1d
    coeffs = state.interior_coeffs(var)[:, :, level, :]
    vals = np.einsum("qm,xym->xyq", vander.phi, coeffs)
    lam, th = element_node_coords(mesh, quad.nodes)
    ref = np.broadcast_to(reference_fn(lam[:, None, :, None], th[None, :, None, :]),
                          (mesh.nx, mesh.ny, n, n)).reshape(mesh.nx, mesh.ny, n * n)
    w2 = np.outer(quad.weights, quad.weights).reshape(-1)
    w_rows = (w2.reshape(n, n)[None, :, :] * np.cos(th)[:, None, :]).reshape(mesh.ny, n * n)
    err = _ordered_sum(mesh.determ * np.einsum("xyq,yq->xy", (vals - ref) ** 2, w_rows))
    norm = _ordered_sum(mesh.determ * np.einsum("xyq,yq->xy", ref**2, w_rows))
    e = math.sqrt(max(err, 0.0))
    return e / math.sqrt(max(norm, 1e-300)) if relative else e


def convergence_rate(eps1: float, h1: float, eps2: float, h2: float) -> float:
    if min(eps1, eps2, h1, h2) <= 0.0:
        raise ValueError("errors and mesh sizes must be positive")
    if h1 == h2:
        raise ValueError("mesh sizes must differ")
    return (math.log(eps1) - math.log(eps2)) / (math.log(h1) - math.log(h2))
